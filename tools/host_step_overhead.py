"""Wall time per spattn_step_host call at a tiny and the c2 shape (profiling helper)."""
import time, torch, sys
sys.path.insert(0, ".")
import paper_2505_22296_b200 as P
for L, H, Hkv in ((256, 32, 8), (32768, 32, 8)):
    mk = lambda h: torch.randn(1, L, h, 128).bfloat16().pin_memory()
    q, k, v, do = mk(H), mk(Hkv), mk(Hkv), mk(H)
    for _ in range(3):
        P.attention_step_host("oracle", q, k, v, do)
    torch.cuda.synchronize()
    n = 20 if L < 1000 else 5
    t = time.perf_counter()
    for _ in range(n):
        P.attention_step_host("oracle", q, k, v, do)
    torch.cuda.synchronize()
    print(L, "wall ms per step", (time.perf_counter() - t) / n * 1e3)
