set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout -s KILL 600 python -m pytest tests -m gpu -q -x -p no:cacheprovider --timeout 200 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -30 gpurun_out/pytest_gpu.log
bash tools/hang_matrix.sh > gpurun_out/hang.log 2>&1; cat gpurun_out/hang.log | head -40
timeout -s KILL 400 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?"; tail -3 gpurun_out/bench.log
