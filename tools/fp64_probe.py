"""Measure the FP64 DADD/DMUL issue rate of this B200 (roofline denominator)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2109_00857_b200 import _lib


def fp64_peak(iters=4096, reps=5):
    L = _lib.load()
    sink = torch.zeros(1, dtype=torch.float64, device="cuda")
    sm = torch.cuda.get_device_properties(0).multi_processor_count
    blocks = sm * 8
    s = _lib.stream_ptr()
    L.fm_fp64_probe(sink.data_ptr(), blocks, 64, s)
    torch.cuda.synchronize()
    best = 0.0
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        _lib.check(L.fm_fp64_probe(sink.data_ptr(), blocks, iters, s), "probe")
        e1.record()
        torch.cuda.synchronize()
        ops = blocks * 256 * iters * 8 * 2  # 8 chains x (DMUL + DADD)
        best = max(best, ops / (e0.elapsed_time(e1) / 1e3))
    return best


if __name__ == "__main__":
    print(json.dumps({"fp64_ops_per_s": fp64_peak()}))
