for r in 1 2; do for n in 1 2 4; do echo -n "NACC=$n "; DFK_NACC=$n timeout 120 python tools/ab_time.py | tail -1; done; done
DFK_LIB=abtest/libdfk_4930b82.so timeout 120 python tools/ab_time.py | tail -1
