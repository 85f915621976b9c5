timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "golden or batch_sweep or ragged or baseline_config or llama8b_full" 2>&1 | tail -4
export AB_SHAPES=4096x1792,5120x3456,8192x3584,5120x6912,4096x3584
AB_TAG=base python tools/shard_ab.py
AB_TAG=dsk2 AB_CFG=block_kernel=1,dynamic_sched=1,s1_split_k=2 python tools/shard_ab.py
AB_TAG=dsk4 AB_CFG=block_kernel=1,dynamic_sched=1,s1_split_k=4 python tools/shard_ab.py
AB_TAG=dsk2g148 DFK_GRID=148 AB_CFG=block_kernel=1,dynamic_sched=1,s1_split_k=2 python tools/shard_ab.py
AB_TAG=dsk4g148 DFK_GRID=148 AB_CFG=block_kernel=1,dynamic_sched=1,s1_split_k=4 python tools/shard_ab.py
AB_TAG=base python tools/shard_ab.py
