"""Writes tests/golden/c1_decode.txt: the FP64 oracle (oracle/attention.py) on the C1 problem drawn
by synth/lcg.py — the expected values of the plain-C GPU client (tests/c/abi_gpu.c).  Calls only
oracle/ and the input generator.  Format: 32 lines "b h lse" then 4096 lines of out in [B, Hq, D]
order, %.17g."""
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import attention as oa  # noqa: E402
from synth import lcg  # noqa: E402


def golden_text() -> str:
    lens, indptr, indices, num_pages, q, k, v = lcg.c1_problem()
    out, lse = oa.paged_decode_attention(q, k, v, indptr, indices, lens, 2)
    lines = [f"{b} {h} {lse[b, h]:.17g}" for b in range(4) for h in range(8)]
    lines += [f"{x:.17g}" for x in out.reshape(-1)]
    return "\n".join(lines) + "\n"


if __name__ == "__main__":
    with open(os.path.join(HERE, "c1_decode.txt"), "w") as f:
        f.write(golden_text())
