set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
nvidia-smi topo -m | head -5
lscpu | grep -i "model name"
nproc
timeout 300 python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 tools/nccl_same_gpu_probe.py 2>&1 | tail -20
timeout 300 python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 tools/tp_ipc_probe.py 2>&1 | tail -5
timeout 1200 python -m pytest tests -x -q -m gpu 2>&1 | tail -15
