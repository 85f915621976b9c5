set -x
export DFK_TEST_TMP=/tmp
timeout 600 compute-sanitizer --tool memcheck --print-limit 20 tests/cpp/test_deepfusion_gpu 2>&1 | tail -60
timeout 600 tests/cpp/test_tuner_gpu 2>&1 | tail -30
timeout 900 python -m pytest tests/test_gpu_graph_and_tp_contract.py tests/test_gpu_tp_multiproc.py tests/test_cpp_shim.py -q 2>&1 | tail -30
