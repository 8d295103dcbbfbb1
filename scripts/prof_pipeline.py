"""Development: host-side profile of the pipeline bench loop (one rank, N = 1): where the
per-step host time goes (cProfile of bench.run_pipeline_arm, the l4 arm)."""
import cProfile
import os
import pstats
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.distributed as dist

import bench
from paper_2512_19179_b200 import pipeline


def main():
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{bench.free_port()}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    stages, _ = pipeline.plan_stages(1, seed=0)
    device = torch.device("cuda", 0)
    kw = dict(precopy_lead=8, policy="bidask", rebalance_every=10)
    bench.run_pipeline_arm(stages, 10, 5, 0, 1, device, **kw)      # warm-up (module loads, allocator)
    pr = cProfile.Profile()
    pr.enable()
    t = bench.run_pipeline_arm(stages, 40, 5, 0, 1, device, **kw)
    pr.disable()
    print(f"host ms/step {t['host_ms_per_step']:.3f}, device elapsed ms/step {t['elapsed_ms'] / 40:.3f}, "
          f"busy ms/step {t['busy_ms'] / 40:.3f}")
    pstats.Stats(pr).sort_stats("tottime").print_stats(25)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
