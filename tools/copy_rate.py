"""Achieved HBM rate of the row copier (shard_rows: one copy-task launch) at several sizes and
row widths (profiling helper).  python tools/copy_rate.py"""
import sys

import torch

sys.path.insert(0, ".")
import paper_2505_22296_b200 as P  # noqa: E402

for L, heads in ((131072, 32), (32768, 32), (32768, 4), (4096, 32), (4096, 4)):
    x = torch.randn(1, L, heads, 128, device="cuda").bfloat16()
    for _ in range(3):
        P.shard_rows(x, "zigzag", 2, 0)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 20
    a.record()
    for _ in range(n):
        P.shard_rows(x, "zigzag", 2, 0)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / n
    moved = 2 * x.numel() * 2 / 2  # read + write of half the rows
    print(f"rows {L // 2} x {heads * 256} B: {moved / 1e6:.1f} MB moved in {ms * 1e3:.1f} us = "
          f"{moved / ms / 1e6:.0f} GB/s")
