export PYTHONFAULTHANDLER=1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()"; echo smoke rc=$?
timeout 2400 python -m pytest tests -q -m gpu -rf --timeout 900 > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -8 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu --no-decode --sweep 1,16,64 --tp-emulate > gpurun_out/bench_emul2.json 2> gpurun_out/bench_emul2.err; echo emul rc=$?
tail -c 1500 gpurun_out/bench_emul2.json; tail -5 gpurun_out/bench_emul2.err
timeout 100 python bench.py --gpus 2 --steps 3; echo "gpus2-on-1 rc=$?"
