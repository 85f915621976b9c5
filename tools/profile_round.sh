#!/bin/bash
# One GPU call: bench line, ncu launch list of a short bench, ncu --set full of
# the default (block) kernel at every batch of the sweep.  Outputs under
# gpurun_out/ (summarise with tools/ncu_summary.py).
set -u
OUT=${OUT:-gpurun_out}
mkdir -p $OUT
NCU=/usr/local/cuda/bin/ncu
if [ -z "${NOBENCH:-}" ]; then
timeout -s KILL 600 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"
tail -c 3000 $OUT/bench.json
timeout -s KILL 900 $NCU --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
  --log-file $OUT/launches.csv python bench.py --steps 2 --warmup 3 --no-tune --no-cpu --sets 2 \
  --no-decode --no-tp-shards > $OUT/bench_ncu.log 2>&1; echo "ncu launches rc=$?"
fi
for B in ${SWEEP:-1 2 4 8 16 32 64}; do
  timeout -s KILL 300 $NCU --set full --clock-control none --import-source on -k regex:stream_kernel \
    -s 4 -c 1 -f -o $OUT/block_B${B} python tools/profile_block.py --B $B > $OUT/ncu_B$B.log 2>&1
  echo "ncu full B=$B rc=$?"
done
