run() { echo -n "$* :: "; env "$@" timeout 120 python tools/ab_time.py 2>&1 | tail -1; }
for r in 1 2; do
run X=0
for k in 4 8 12 16 20 24; do run DFK_PF_KB=$k; done
done
