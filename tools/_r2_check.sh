set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
lscpu | grep -i "model name"; nproc
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
timeout 2400 python -m pytest tests -q -m gpu -rf --timeout 900 > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -30 gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$?
tail -c 3000 gpurun_out/bench.json
