"""Read-bandwidth probe (development evidence): the HBM read ceiling a streaming kernel can
reach on this B200, for comparison with decode_kernel's achieved GB/s (the roofline
denominator stays MEASURED_PEAKS.json's copy figure).  Needs scripts/readbw.so
(scripts/build_readbw.sh)."""
import ctypes
import json
import os

import torch

HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    lib = ctypes.CDLL(os.path.join(HERE, "readbw.so"))
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    res = {}
    sink = torch.zeros(1, dtype=torch.int64, device="cuda")
    for gb in (1, 4):
        n = gb << 30
        buf = torch.empty(n, dtype=torch.uint8, device="cuda")
        buf.random_(0, 255)
        st = torch.cuda.current_stream().cuda_stream

        def t(fn, reps=20):
            for _ in range(3):
                fn()
            torch.cuda.synchronize()
            best = 1e9
            for _ in range(reps):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                fn()
                b.record()
                b.synchronize()
                best = min(best, a.elapsed_time(b))
            return round(n / (best / 1e3) / 1e9, 1)

        for mult, block in ((4, 512), (8, 256), (16, 256), (32, 256)):
            res[f"ldg_{gb}GB_grid{mult}x_b{block}"] = t(lambda: lib.probe_ldg(
                ctypes.c_void_p(buf.data_ptr()), ctypes.c_size_t(n), mult * sms, block,
                ctypes.c_void_p(sink.data_ptr()), ctypes.c_void_p(st)))
        for ctas, kb in ((1, 128), (2, 64), (2, 96), (3, 64)):
            res[f"tma_{gb}GB_{ctas}cta_{kb}KB"] = t(lambda: lib.probe_tma(
                ctypes.c_void_p(buf.data_ptr()), ctypes.c_size_t(n), ctas * sms, kb,
                ctypes.c_void_p(sink.data_ptr()), ctypes.c_void_p(st)))
        c = torch.empty(n // 2, dtype=torch.uint8, device="cuda")
        res[f"copy_{gb}GB_rw"] = t(lambda: c.copy_(buf[: n // 2]))  # bytes read + written = n
        del buf, c
        torch.cuda.empty_cache()
    print(json.dumps(res))


if __name__ == "__main__":
    main()
