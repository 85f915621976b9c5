#!/bin/bash
# One GPU call: bench line, ncu launch list of a short bench, ncu --set full of
# the default (block) kernel at every batch of the sweep, summarised on the box
# (tools/ncu_summary.py) so that only small files come back: block_traffic.json
# (bench.py's roofline.traffic), launches.md/.csv, raw pages of B = 1/16/64.
# The .ncu-rep files are deleted after summarising (they exceed gpurun's 64 MiB
# transfer limit together).  Outputs under $OUT (default gpurun_out/prof).
set -u
OUT=${OUT:-gpurun_out/prof}
mkdir -p $OUT
NCU=/usr/local/cuda/bin/ncu
if [ -z "${NOBENCH:-}" ]; then
timeout -s KILL 600 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"
tail -c 3000 $OUT/bench.json
timeout -s KILL 900 $NCU --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
  --log-file $OUT/launches.csv python bench.py --steps 2 --warmup 3 --no-tune --no-cpu --sets 2 \
  --no-decode --no-tp-shards > $OUT/bench_ncu.log 2>&1; echo "ncu launches rc=$?"
# the same command's timed region only (bench.py brackets it with
# cudaProfilerStart/Stop under DFK_PROFILE_TIMED=1): the kernels of the steps
DFK_PROFILE_TIMED=1 timeout -s KILL 900 $NCU --profile-from-start off --metrics gpu__time_duration.sum \
  --clock-control none --csv --log-file $OUT/launches_timed.csv python bench.py --steps 2 --warmup 3 \
  > $OUT/bench_ncu_timed.log 2>&1; echo "ncu timed launches rc=$?"
fi
for B in ${SWEEP:-1 2 4 8 16 32 64}; do
  timeout -s KILL 300 $NCU --set full --clock-control none --import-source on -k regex:stream_kernel \
    -s 4 -c 1 -f -o $OUT/block_B${B} python tools/profile_block.py --B $B > $OUT/ncu_B$B.log 2>&1
  echo "ncu full B=$B rc=$?"
done
python tools/ncu_summary.py traffic $OUT/block_traffic.json $OUT/block_B*.ncu-rep > $OUT/summary.log 2>&1
[ -f $OUT/launches.csv ] && python tools/ncu_summary.py launches $OUT/launches.md $OUT/launches.csv >> $OUT/summary.log 2>&1
[ -f $OUT/launches_timed.csv ] && python tools/ncu_summary.py launches $OUT/launches_timed.md $OUT/launches_timed.csv >> $OUT/summary.log 2>&1
for B in 1 16 64; do
  [ -f $OUT/block_B$B.ncu-rep ] && $NCU -i $OUT/block_B$B.ncu-rep --page raw --csv > $OUT/block_B${B}_raw.csv 2>/dev/null
done
[ -z "${KEEP_REPS:-}" ] && rm -f $OUT/*.ncu-rep
du -sh $OUT
