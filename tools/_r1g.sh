timeout -s KILL 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider --timeout 300 2>&1 | tail -3
timeout -s KILL 900 python tools/tp_shard_sweep.py --specs "default;variant=1;tune" --json gpurun_out/tp_shard4.json > gpurun_out/tp_shard4.txt 2>&1; tail -3 gpurun_out/tp_shard4.txt
timeout -s KILL 600 python bench.py > gpurun_out/bench4.json 2> gpurun_out/bench4.err; echo "bench rc=$?"; tail -c 2500 gpurun_out/bench4.json
