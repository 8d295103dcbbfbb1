"""Development: the end-to-end (host buffers) measurement of bench.py alone."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench

for name in ("c2", "c3"):
    spec = bench.WORKLOADS[name]
    wl = bench.Workload(name, spec["lens"](), spec["shape"])
    ms, h2d, d2h = bench.time_e2e(wl, 20, 3)
    print(name, f"{ms / 20 * 1e3:.1f} us/step, {wl.bytes_kv / (ms / 20 / 1e3) / 1e9:.0f} GB/s, H2D {h2d} B, D2H {d2h} B")
