"""The driver's bench.py contract, checked on CPU: the reference arm
(`--impl reference`, the reference's own CPU run_fused from oracle/_ref) prints
one JSON line with the keys the driver reads, and `--gpus N` refuses to run on
fewer visible GPUs instead of silently measuring one."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run_bench(*args, timeout=300):
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args],
                          capture_output=True, text=True, timeout=timeout, cwd=ROOT)


@pytest.mark.skipif(not os.path.exists(os.path.join(ROOT, "oracle", "_ref")),
                    reason="oracle/_ref not built")
def test_reference_arm_prints_one_contract_line():
    r = run_bench("--impl", "reference", "--steps", "1", "--warmup", "3")
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
              "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["steps"] == 1 and d["warmup"] == 3
    assert d["value"] > 0 and d["higher_is_better"] is True
    assert d["e2e"]["value"] == d["value"] and d["e2e"]["unit"] == d["unit"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    cb = d["cpu_baseline"]
    assert cb["kind"] in ("reference", "port") and cb["cores"] >= 1 and cb["value"] == d["value"]
    assert d["config"]["workload"].startswith("Llama-3.1-8B MLP")


def test_gpus_beyond_visible_devices_refused():
    import ctypes
    try:  # how many GPUs this host shows (none in the build container)
        n = ctypes.c_int(0)
        ctypes.CDLL("libcudart.so").cudaGetDeviceCount(ctypes.byref(n))
        visible = n.value
    except OSError:
        visible = 0
    want = max(2, visible + 1)  # (--gpus 1 on a GPU-less host just fails to find a device)
    r = run_bench("--gpus", str(want), "--steps", "1", "--warmup", "3", timeout=120)
    assert f"needs {want} visible GPUs" in (r.stdout + r.stderr), (r.stdout, r.stderr)
    assert not [ln for ln in r.stdout.splitlines() if ln.startswith('{"metric"')]
