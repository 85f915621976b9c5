timeout -s KILL 400 python -m pytest tests/test_gpu_parity.py -q -x -k "decode" -p no:cacheprovider --timeout 200 2>&1 | tail -15
timeout -s KILL 400 python bench.py --no-cpu --steps 10 > gpurun_out/bench_dec.json 2> gpurun_out/bench_dec.err; echo "bench rc=$?"; tail -c 1500 gpurun_out/bench_dec.json; tail -5 gpurun_out/bench_dec.err
