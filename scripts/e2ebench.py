"""Development: the end-to-end (host buffers) measurement of bench.py alone."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench

for name in ("c2", "c3"):
    spec = bench.WORKLOADS[name]
    wl = bench.Workload(name, spec["lens"](), spec["shape"])
    for ns in (1, 2):
        for bf in (False, True):
            ms, h2d, d2h = bench.time_e2e(wl, 20, 3, n_streams=ns, out_bf16=bf)
            print(name, f"streams {ns} out {'bf16' if bf else 'f32'}: {ms / 20 * 1e3:.1f} us/step, "
                  f"{wl.bytes_kv / (ms / 20 / 1e3) / 1e9:.0f} GB/s, H2D {h2d} B, D2H {d2h} B")
