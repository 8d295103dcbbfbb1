#!/bin/bash
# Development check of the N-rank pipeline harness on ONE GPU: all ranks share cuda:0 and the
# page transport goes through gloo (host-staged).  The driver's real runs use NCCL, 1 GPU/rank.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
for n in 2 4; do
  L4_FORCE_DEVICE=0 L4_PIPE_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n \
    --master-addr 127.0.0.1 --master-port $((29500 + n)) bench.py --gpus $n --steps 30 --warmup 5 \
    > gpurun_out/multirank_$n.log 2>&1
  echo "== n=$n rc=$?"; tail -2 gpurun_out/multirank_$n.log | cut -c1-3000
done
