for r in 1 2; do
for l in abtest/libdfk_4930b82.so abtest/libdfk_notpp.so; do
  DFK_LIB=$l timeout 120 python tools/ab_time.py 2>&1 | tail -1
done; done
