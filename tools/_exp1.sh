S="block:dynamic_sched=1;block:dynamic_sched=1,kbs=4,s1_stages=2;block:dynamic_sched=1,kbs=3,s1_stages=3;block:dynamic_sched=1,kbs=2,s1_stages=3;block:dynamic_sched=1,kbs=2,s1_stages=4;block:dynamic_sched=1,kbs=1,s1_stages=9;block:dynamic_sched=1,kbs=3,s1_stages=2"
timeout 300 python tools/sweep_configs.py --batches 1,16,32,64 --what none --sets 4 --reps 30 --specs "$S"
S2="s1:kbs=4;s1:kbs=3,s1_stages=3;s1:kbs=2,s1_stages=4;s1:kbs=3,s1_stages=2;s1:s1_ctas=148;s1:kbs=2,s1_ctas=148"
timeout 300 python tools/sweep_configs.py --batches 1,64 --what none --sets 4 --reps 30 --specs "$S2"
