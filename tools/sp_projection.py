"""Single-GPU measurement of the SP engines at BASELINE configs c1-c5, projected to N GPUs.

This run has one B200, so the multi-GPU configs are measured as follows (and labelled
"projected"): all `sp` ranks of the engine run on one GPU through the loopback fabric, the GPU
time of one fwd+bwd of the whole layer (T_all, CUDA events) is split by each rank's exact share
of the attention work (admitted pairs x heads, from the engine's own flop counters), and the
busiest rank's per-step communication (this implementation's measured send-side bytes) is added
at the measured NVLink peer bandwidth (770 GB/s per direction, B200_PROFILING.md) without
overlap — an upper bound on the step time:
    t_rank = T_all * flops_busiest / flops_total + bytes_busiest / 770 GB/s
    tokens/s = L / t_rank
    python tools/sp_projection.py [--quick] > profiles/r1_sp_projection.md
"""
import json
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import paper_2505_22296_b200 as P  # noqa: E402

NVLINK = 770e9
HBM = 6.5e12  # measured copy bandwidth order (MEASURED_PEAKS.json hbm_gbs)


def c5_docs(total=262144, lo=1024, hi=65536):
    """Rng(5).uniform_int(1024, 65536) until the running sum would exceed 262144;
    the final document absorbs the remainder."""
    import seqpar_oracle as O

    rng, docs, s = O.Rng(5), [], 0
    while True:
        n = rng.uniform_int(lo, hi)
        if s + n > total:
            break
        docs.append(n)
        s += n
    if total - s >= lo or not docs:
        docs.append(total - s)
    else:
        docs[-1] += total - s
    return docs


def run(engine, sp, L, H, Hkv, d, docs=None, u=0, r=0, reps=2, layout="auto"):
    g = torch.Generator(device="cuda").manual_seed(0)
    q = torch.randn(1, L, H, d, device="cuda", generator=g).bfloat16().requires_grad_(True)
    k = torch.randn(1, L, Hkv, d, device="cuda", generator=g).bfloat16().requires_grad_(True)
    v = torch.randn(1, L, Hkv, d, device="cuda", generator=g).bfloat16().requires_grad_(True)
    dout = torch.randn(1, L, H, d, device="cuda", generator=g).bfloat16()
    fab = P.Fabric(sp)
    times = []
    for rep in range(reps + 1):
        fab.reset_stats()
        q.grad = k.grad = v.grad = None
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        out = P.engine_attention(engine, q, k, v, sp, docs=docs, fabric=fab, ulysses_degree=u,
                                 ring_degree=r, layout=layout)
        out.backward(dout)
        torch.cuda.synchronize()
        if rep:  # first run warms up
            times.append(time.perf_counter() - t0)
    # the loopback driver synchronises every rank stream inside each call, so host wall time of
    # the call pair is the GPU time of the layer (plus sharding/gathering, excluded below)
    flops = [fab.flops(i) for i in range(sp)]
    nbytes = [fab.total_bytes(i) for i in range(sp)]
    return min(times), flops, nbytes


def shard_overhead(L, H, Hkv, d, sp):
    """Host-side shard/gather of the loopback wrapper (not part of the layer): measured with a
    no-op of the same tensor traffic."""
    x = torch.randn(1, L, H, d, device="cuda").bfloat16()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(2):
        shards = [P.shard_rows(x, "naive", sp, i) for i in range(sp)]
        P.gather_rows(shards, "naive", sp)
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / 2 * (2 + 2 * Hkv / H + 2)  # q,k,v,dout in; out,dq,dk,dv out


def main():
    quick = "--quick" in sys.argv
    scen = [
        ("c1", "ulysses", 2, 4096, 8, 8, 64, None, 0, 0),
        ("c2", "ulysses", 1, 32768, 32, 8, 128, None, 0, 0),
        ("c2", "ulysses", 2, 32768, 32, 8, 128, None, 0, 0),
        ("c2", "ulysses", 4, 32768, 32, 8, 128, None, 0, 0),
        ("c2", "ulysses", 8, 32768, 32, 8, 128, None, 0, 0),
        ("c3", "dummy_head", 8, 65536, 28, 4, 128, None, 0, 0),
        ("c3", "xtuner", 8, 65536, 28, 4, 128, None, 0, 0),
        # USP with an inner Ulysses degree that divides the 28 heads: no dummy heads, no idle rank
        ("c3", "usp", 8, 65536, 28, 4, 128, None, 4, 2),
        ("c3", "usp", 8, 65536, 28, 4, 128, None, 2, 4),
        ("c4", "ring", 2, 131072, 32, 8, 128, None, 0, 0),
        ("c4", "ring", 4, 131072, 32, 8, 128, None, 0, 0),
        ("c4", "ring", 8, 131072, 32, 8, 128, None, 0, 0),
        ("c4", "ulysses", 8, 131072, 32, 8, 128, None, 0, 0),
        ("c4", "usp", 8, 131072, 32, 8, 128, None, 2, 4),
        ("c5", "ulysses", 8, 262144, 32, 8, 128, "docs", 0, 0),
        ("c5", "ring", 8, 262144, 32, 8, 128, "docs", 0, 0),
    ] + [("c5", "ring", 8, 262144, 32, 8, 128, "docs", 0, 0, f"zigzag:{b}")
         for b in next((a.split("=", 1)[1] for a in sys.argv if a.startswith("--c5-blocks=")), "16").split(",")]
    only = [a.split("=", 1)[1] for a in sys.argv if a.startswith("--only=")]
    if only:
        scen = [x for x in scen if x[0] in only[0].split(",")]
    scen = [x if len(x) == 11 else x + ("auto",) for x in scen]
    if quick:
        scen = [s[:3] + (min(s[3], 16384),) + s[4:] for s in scen if s[0] in ("c1", "c3", "c4")][:5]
    rows = []
    for name, engine, sp, L, H, Hkv, d, docs, u, r, layout in scen:
        dl = c5_docs(L) if docs == "docs" else None
        t_all, flops, nbytes = run(engine, sp, L, H, Hkv, d, dl, u, r, layout=layout)
        t_all -= shard_overhead(L, H, Hkv, d, sp) if sp > 1 else 0.0
        busiest = max(range(sp), key=lambda i: flops[i])
        share = flops[busiest] / max(1, sum(flops))
        t_comp = t_all * share
        t_comm = nbytes[busiest] / NVLINK
        t_rank = t_comp + t_comm
        # overlap-aware ring estimate (r2 ring engine): the k|v hops of the next step and the
        # dk|dv hop of the previous one travel during a step's kernel; exposed are the hops that
        # outlast a step, the sp-1 dk|dv adds (an HBM pass: 12 bytes per kv element) and the
        # home-coming dk|dv hop
        t_ovl = t_rank
        if engine == "ring" and sp > 1:
            X = L // sp * Hkv * d
            t_fwd_step, t_bwd_step = t_comp * 4 / 14 / sp, t_comp * 10 / 14 / sp
            kv_hop, g_hop = 2 * X * 2 / NVLINK, 2 * X * 4 / NVLINK
            exposed = (sp - 1) * max(0.0, kv_hop - t_fwd_step)
            exposed += (sp - 1) * max(0.0, kv_hop + g_hop - t_bwd_step)
            exposed += (sp - 1) * 3 * 2 * X * 4 / HBM + g_hop
            t_ovl = t_comp + exposed
        real = 14 * d * H * (L * (L + 1) // 2) if dl is None else sum(14 * d * H * n * (n + 1) // 2 for n in dl)
        rows.append(dict(config=name, engine=engine if layout == "auto" else f"{engine} ({layout})", sp=sp, L=L, heads=f"{H}/{Hkv}", d=d,
                         docs=len(dl) if dl else 0, t_all_ms=t_all * 1e3,
                         busiest_share=share, t_compute_ms=t_comp * 1e3,
                         bytes_busiest=nbytes[busiest], t_comm_ms=t_comm * 1e3,
                         t_step_ms=t_rank * 1e3, tokens_per_s=L / t_rank,
                         t_step_overlap_ms=t_ovl * 1e3, tokens_per_s_overlap=L / t_ovl,
                         executed_flops=sum(flops), algorithmic_flops=real,
                         achieved_tflops_1gpu=sum(flops) / t_all / 1e12))
        print(json.dumps(rows[-1]), file=sys.stderr, flush=True)
    print("| config | engine | SP | L | heads q/kv | docs | T_all 1-GPU (ms) | busiest share | "
          "t_compute (ms) | bytes/rank (MB) | t_comm@770GB/s (ms) | projected step (ms) | "
          "projected tokens/s | overlap-aware step (ms) | 1-GPU TFLOP/s (executed) |")
    print("|---|---|---|---|---|---|---|---|---|---|---|---|---|---|---|")
    for x in rows:
        print(f"| {x['config']} | {x['engine']} | {x['sp']} | {x['L']} | {x['heads']} | {x['docs']} | "
              f"{x['t_all_ms']:.1f} | {x['busiest_share']:.3f} | {x['t_compute_ms']:.2f} | "
              f"{x['bytes_busiest'] / 1e6:.1f} | {x['t_comm_ms']:.2f} | {x['t_step_ms']:.2f} | "
              f"{x['tokens_per_s']:.3e} | {x['t_step_overlap_ms']:.2f} | {x['achieved_tflops_1gpu']:.0f} |")
    json.dump(rows, open(os.path.join(ROOT, "profiles", "sp_projection.json"), "w"), indent=1)


if __name__ == "__main__":
    main()
