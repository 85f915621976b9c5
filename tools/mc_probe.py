"""Probe: is CUDA multicast (NVLS) available on this box?"""
import ctypes as C
cu = C.CDLL("libcuda.so.1")
cu.cuInit(0)
dev = C.c_int()
cu.cuDeviceGet(C.byref(dev), 0)
v = C.c_int()
# CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED = 132
r = cu.cuDeviceGetAttribute(C.byref(v), 132, dev)
print("cuDeviceGetAttribute(MULTICAST_SUPPORTED) ->", r, "value", v.value)
n = C.c_int()
cu.cuDeviceGetCount(C.byref(n))
print("visible devices", n.value)
