#!/bin/bash
# Development check of the N-rank pipeline harness on ONE GPU: all ranks share cuda:0 and the
# default process group is gloo.  Page transport: TRANSPORTS="gloo ipc" — host-staged two-sided
# (gloo) and the one-sided CUDA-IPC push (DeviceOps.setup_ipc).  The driver's real runs use
# NCCL with one GPU per rank.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
for tr in ${TRANSPORTS:-gloo ipc}; do
  for n in ${NS:-2 4}; do
    tp=nccl; [ "$tr" = ipc ] && tp=ipc
    L4_FORCE_DEVICE=0 L4_PIPE_BACKEND=gloo L4_PIPE_TRANSPORT=$tp timeout 900 python -m torch.distributed.run --nnodes=1 \
      --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29500 + n)) bench.py --gpus $n --steps 30 --warmup 5 \
      > gpurun_out/multirank_${tr}_$n.log 2>&1
    echo "== transport=$tr n=$n rc=$?"; tail -1 gpurun_out/multirank_${tr}_$n.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); p=d['pipeline']
print({k:(round(v['kv_gbs']), round(v['tokens_per_s']), round(v['mean_step_latency_ms'],3), v['migrations'], v['migrated_bytes']) for k,v in p.items()})" 2>&1 | tail -1
  done
done
