"""Per-group timeline of spattn_step_host at the bench's c4 shape (SPATTN_STEP_TRACE=1 prints
it to stderr; profiling helper).  SPATTN_STEP_TRACE=1 python tools/step_trace.py [L]"""
import sys

import torch

sys.path.insert(0, ".")
import paper_2505_22296_b200 as P  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 131072
mk = lambda h: torch.randn(1, L, h, 128).bfloat16().pin_memory()  # noqa: E731
q, k, v, do = mk(32), mk(8), mk(8), mk(32)
for _ in range(2):
    P.attention_step_host("ring", q, k, v, do)
torch.cuda.synchronize()
