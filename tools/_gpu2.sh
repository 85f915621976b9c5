set -x
python -c "import __graft_entry__ as g; g.smoke()"
timeout 900 python -m pytest tests/test_gpu_graph_and_tp_contract.py tests/test_gpu_tp_multiproc.py -x -q 2>&1 | tail -30
timeout 1200 python -m pytest tests -x -q -m gpu 2>&1 | tail -15
