#!/bin/bash
# 4-GPU round trip: the NCCL tests at 4 ranks, C2 weak scaling, C5 restore, the T shard x4
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
nvidia-smi topo -m > gpurun_out/topo_n4.txt 2>&1
timeout 900 python -m pytest tests/test_multi_gpu.py -m gpu -q 2>&1 | tail -3
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
timeout 900 $R --master-port 29611 bench.py --gpus 4 --steps 20 --warmup 5 > gpurun_out/m_C2_n4.json 2> gpurun_out/m_C2_n4.err; echo "C2 n=4 rc=$?"
timeout 900 $R --master-port 29612 bench.py --workload C5 --gpus 4 --steps 10 --warmup 3 > gpurun_out/m_C5_n4.json 2> gpurun_out/m_C5_n4.err; echo "C5 n=4 rc=$?"
timeout 1500 $R --master-port 29613 bench.py --workload T --gpus 4 --steps 10 --warmup 3 > gpurun_out/m_T_n4.json 2> gpurun_out/m_T_n4.err; echo "T n=4 rc=$?"
# C3 (Criteo-TB-shaped, 4-bit adaptive greedy) row-sharded over 2 and 4 GPUs, and 1 for the ratio
timeout 900 python bench.py --workload C3 --steps 10 --warmup 3 --no-cpu > gpurun_out/m_C3_n1.json 2> gpurun_out/m_C3_n1.err; echo "C3 n=1 rc=$?"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29614 bench.py --workload C3 --gpus 2 --steps 10 --warmup 3 > gpurun_out/m_C3_n2.json 2> gpurun_out/m_C3_n2.err; echo "C3 n=2 rc=$?"
timeout 900 $R --master-port 29615 bench.py --workload C3 --gpus 4 --steps 10 --warmup 3 > gpurun_out/m_C3_n4.json 2> gpurun_out/m_C3_n4.err; echo "C3 n=4 rc=$?"
