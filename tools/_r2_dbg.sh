export AB_SHAPES=4096x1792,5120x3456,8192x3584,5120x6912
AB_TAG=base python tools/shard_ab.py
AB_TAG=static AB_CFG=block_kernel=1 python tools/shard_ab.py
AB_TAG=sk2 AB_CFG=block_kernel=1,s1_split_k=2 python tools/shard_ab.py
AB_TAG=sk4 AB_CFG=block_kernel=1,s1_split_k=4 python tools/shard_ab.py
AB_TAG=sk8 AB_CFG=block_kernel=1,s1_split_k=8 python tools/shard_ab.py
AB_TAG=nopdl AB_CFG=block_kernel=1,dynamic_sched=1,pdl=0 python tools/shard_ab.py
