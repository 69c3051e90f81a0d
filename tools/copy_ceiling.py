#!/usr/bin/env python
"""HBM copy ceiling at the gather's size: back-to-back device copies of one Falcon-7B
block's bf16 buffer (207,071,232 elements = 414 MB read + 414 MB written per copy), the
shape of an N = 1 forward / backward gather, vs the 1 Gi-element copy MEASURED_PEAKS.json
uses.  torch `copy_` (same-dtype contiguous: the driver's D2D memcpy) and an elementwise
SM kernel (`mul(src, 1)`), CUDA events around back-to-back copies (34 = one step's
gathers at the block size), best of 5."""
import json

import torch


def rate(fn, nbytes, reps=34, rounds=5):
    best = 0.0
    for _ in range(rounds):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record()
        for _ in range(reps):
            fn()
        b.record()
        torch.cuda.synchronize()
        best = max(best, 2 * nbytes * reps / (a.elapsed_time(b) * 1e-3) / 1e9)
    return round(best, 1)


def main():
    out = {}
    for name, n in (("falcon7b_block", 207_071_232), ("1Gi", 1 << 30)):
        src = torch.empty(n, dtype=torch.bfloat16, device="cuda").normal_()
        dst = torch.empty_like(src)
        nbytes = n * 2
        reps = 34 if n < (1 << 30) else 8
        out[name] = {"elements": n, "torch_copy_GBps": rate(lambda: dst.copy_(src), nbytes, reps),
                     "elementwise_kernel_GBps": rate(lambda: torch.mul(src, 1, out=dst), nbytes, reps)}
        del src, dst
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
