#!/bin/bash
# multi-GPU round trip: the NCCL tests, then C2 weak scaling and C5 restore at N GPUs
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
nvidia-smi topo -m > gpurun_out/topo_n$N.txt 2>&1
timeout 900 python -m pytest tests/test_multi_gpu.py -m gpu -q 2>&1 | tail -4
for n in $(seq 2 $N); do
  [ $n -eq 3 ] && continue
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29600+n)) bench.py --gpus $n --steps 20 --warmup 5 > gpurun_out/m_C2_n$n.json 2> gpurun_out/m_C2_n$n.err; echo "C2 n=$n rc=$?"
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29700+n)) bench.py --workload C5 --gpus $n --steps 10 --warmup 3 > gpurun_out/m_C5_n$n.json 2> gpurun_out/m_C5_n$n.err; echo "C5 n=$n rc=$?"
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29800+n)) bench.py --impl reference --gpus $n --steps 2 --warmup 1 > gpurun_out/m_ref_n$n.json 2> gpurun_out/m_ref_n$n.err; echo "ref n=$n rc=$?"
done
timeout 600 python bench.py --workload C5 --steps 10 --warmup 3 > gpurun_out/m_C5_n1.json 2> gpurun_out/m_C5_n1.err; echo "C5 n=1 rc=$?"
