#!/usr/bin/env python
"""SP attention fwd+bwd throughput (BASELINE.json metric) on B200.

Headline workload (BASELINE.json configs[3], the largest config that fits one GPU and the one
north_star quotes its 128K scaling target on): Llama-3-8B attention shape — 32 Q / 8 KV heads,
head_dim 128, causal, seq 131072, bs 1 — as zigzag Ring SP=N over N GPUs (one process per GPU,
NCCL). At N=1 the layer degenerates to the single-GPU attention kernel pair. A step = one
forward + one backward of the layer over the whole sequence (all ranks). The line also carries
`secondary` measurements: Ulysses at the same 128K shape and c2 (32K, Ulysses).

  python bench.py [--gpus N --steps K --warmup W]           # our arm
  python bench.py --impl reference [...]                    # reference CPU arm (oracle/_ref)
Under torchrun: RANK/LOCAL_RANK/WORLD_SIZE from the env, rank 0 prints ONE JSON line.
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import shutil
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "SP attention fwd+bwd tokens/s"
CONFIGS = {
    # name: (heads, kv_heads, head_dim, seq_len, engine)
    "c2": (32, 8, 128, 32768, "ulysses"),
    "c1": (8, 8, 64, 4096, "ulysses"),
    "c3": (28, 4, 128, 65536, "dummy_head"),
    "c4": (32, 8, 128, 131072, "ring"),
}
MODEL_OF = {"c1": "reference parity-grid", "c2": "Llama-3-8B", "c3": "Qwen2.5-7B", "c4": "Llama-3-8B"}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p["bf16_tflops"], p.get("bf16_tflops_sustained", p["bf16_tflops"]), p["hbm_gbs"], "measured"
    except Exception:
        return 1590.0, 1400.0, 6650.0, "fallback"


def causal_pairs(L):
    return L * (L + 1) // 2


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.path = os.path.join(ROOT, "gpurun_out", f"clocks_{os.getpid()}.csv")

    def __enter__(self):
        if shutil.which("nvidia-smi"):
            os.makedirs(os.path.dirname(self.path), exist_ok=True)
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "25"], stdout=self.f,
                stderr=subprocess.DEVNULL)
            time.sleep(0.3)
        return self

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            self.proc.wait()
            self.f.close()

    def summary(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        rows = []
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 9:
                rows.append(parts)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in rows for n, v in zip(names, r[5:9]) if v.lower() == "active"})
        # samples every 25 ms over the barrier + timed steps; the first one precedes the load
        loaded = sm[1:] if len(sm) > 2 else sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(rows)}


# ------------------------------------------------------------------------- CPU baseline
def cpu_reference_sample(heads, kv, d, L, threads=None, engine="ulysses"):
    """Time the UNMODIFIED reference (oracle/_ref/ref_driver, built from /root/reference by
    oracle/Makefile) on a bounded sample of the workload: the config's engine, same head_dim and
    GQA ratio, 8 query heads, seq 2048, over `threads` rank threads (comm.cpp:197-222) — a few
    seconds per sample, so a 20-step reference arm ends in about a minute; extrapolated to the
    full workload by exact causal pair count x heads."""
    ncpu = os.cpu_count() or 1
    sp = 1
    while sp * 2 <= min(ncpu, 8):
        sp *= 2
    if threads:
        sp = threads
    s_heads, s_kv, s_L = 8, max(1, 8 * kv // heads), 2048
    drv = os.path.join(ROOT, "oracle", "_ref", "ref_driver")
    if os.path.exists(drv):
        out = subprocess.run([drv, "bench", engine, str(sp), str(s_L), str(s_heads), str(s_kv),
                              str(d), "1"], capture_output=True, text=True, check=True)
        rec = json.loads(out.stdout.strip().splitlines()[-1])
        secs, kind = rec["s_per_step"], "reference"
    else:  # the plain-C restatement (oracle/liboracle.so) on one thread
        sys.path.insert(0, os.path.join(ROOT, "oracle"))
        import seqpar_oracle as O

        s_L = 1024
        q, k, v, R = O.parity_data(1, s_L, s_heads, s_kv, d)
        t0 = time.perf_counter()
        O.attention_fwd_bwd(q, k, v, R)
        secs, kind, sp = time.perf_counter() - t0, "port", 1
    work_sample = causal_pairs(s_L) * s_heads
    work_full = causal_pairs(L) * heads
    t_full = secs * work_full / work_sample
    return {"value": L / t_full, "unit": "tokens/s", "cores": sp, "kind": kind,
            "extrapolated": True,
            "sample": f"EXTRAPOLATED: {engine if kind == 'reference' else 'oracle'} fwd+bwd, {s_heads}q/{s_kv}kv heads, d={d}, L={s_L}, "
                      f"{sp} rank threads: {secs:.2f} s measured; scaled x{work_full / work_sample:.1f} "
                      f"by causal pairs x heads to L={L}, {heads} heads",
            "sample_seconds": secs}


def run_reference(args, cfg):
    heads, kv, d, L, engine = CONFIGS[cfg]
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    vals, samples = [], []
    if args.warmup > 0:  # one untimed sample warms the page cache and the CPU frequency
        cpu_reference_sample(heads, kv, d, L, engine=engine)
    for _ in range(args.steps):
        r = cpu_reference_sample(heads, kv, d, L, engine=engine)
        vals.append(r["value"])
        samples.append(r)
    v = statistics.median(vals)
    # ms_per_step is the wall time of one timed sample (what this run actually spent per step);
    # value is that sample's throughput extrapolated to the full workload (exact causal pairs x
    # heads), since a full-size CPU step would take hours
    sample_ms = 1000.0 * statistics.median(r["sample_seconds"] for r in samples)
    line = {"metric": METRIC, "value": v, "unit": "tokens/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": sample_ms,
            "extrapolated": {"from": samples[-1]["sample"], "full_step_ms": 1000.0 * L / v},
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (reference Rng uniform(-2,2))", "impl": "reference",
            "config": {"workload": f"{cfg}: {MODEL_OF[cfg]} attention {heads}q/{kv}kv heads "
                                   f"d={d} seq {L} causal bs 1", "engine": engine,
                       "parallelism": f"sp{args.gpus}", "global_batch": 1, "seq_len": L},
            "cpu_baseline": {k: samples[-1][k] for k in ("value", "unit", "cores", "kind", "sample")},
            "e2e": {"value": v, "unit": "tokens/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    line["cpu_baseline"]["value"] = v
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------ our arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c4", choices=sorted(CONFIGS))
    ap.add_argument("--no-secondary", action="store_true")
    ap.add_argument("--engine", default=None)
    ap.add_argument("--seq-len", type=int, default=None)
    ap.add_argument("--family", default="tcgen05", choices=["tcgen05", "mma", "tcgen05_pp", "tcgen05_pair", "tcgen05_q64"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-groups", type=int, default=0,
                    help="kv-head groups of the pipelined host step (0 = library default)")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args, args.config)

    import torch

    import paper_2505_22296_b200 as P
    from paper_2505_22296_b200 import _lib as C

    heads, kv, d, L, engine = CONFIGS[args.config]
    engine = args.engine or engine
    L = args.seq_len or L
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        rc = P.RankContext(sp=world)
        ctx = rc._h
        keep = rc
    else:
        fab = P.Fabric(1)
        ctx = fab.ctxs[0]
        keep = fab
    sp = world
    P.set_kernel_family(args.family)
    mode = "zigzag" if engine == "ring" else "naive"
    lay = C.make_layout(mode, L, sp)
    cfg = C.make_config(heads, kv, d, True)
    lloc = L // sp
    g = torch.Generator(device="cuda").manual_seed(1234 + rank)
    mk = lambda h: torch.randn(1, lloc, h, d, device="cuda", dtype=torch.bfloat16, generator=g)  # noqa
    q, k, v, do = mk(heads), mk(kv), mk(kv), mk(heads)
    out, dq, dk, dv = (torch.empty_like(x) for x in (q, q, k, v))
    lse = torch.empty(1, lloc, heads, device="cuda", dtype=torch.float32)
    stream = torch.cuda.Stream()  # explicit stream: events and kernels share it
    torch.cuda.set_stream(stream)
    C.check(C.lib().spattn_ctx_set_stream(ctx, stream.cuda_stream))
    eid = C.engine_id(engine)

    def step(qp, kp, vp, dop, dqp, dkp, dvp):
        saved = ctypes.c_void_p()
        C.check(C.lib().spattn_fwd(ctx, eid, ctypes.byref(cfg), ctypes.byref(lay), 1, qp, kp, vp,
                                   out.data_ptr(), lse.data_ptr(), None, 0, ctypes.byref(saved)))
        C.check(C.lib().spattn_bwd(ctx, saved, dop, dqp, dkp, dvp))
        C.lib().spattn_saved_free(saved)

    ptrs = (q.data_ptr(), k.data_ptr(), v.data_ptr(), do.data_ptr(), dq.data_ptr(),
            dk.data_ptr(), dv.data_ptr())

    def barrier():
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x):
        if not dist:
            return x
        t = torch.tensor([x], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t.item()

    for _ in range(args.warmup):
        step(*ptrs)
    barrier()
    n0 = C.lib().spattn_launch_count()
    C.check(C.lib().spattn_ctx_reset_stats(ctx))
    C.check(C.lib().spattn_profile_enable(1))
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with Clocks(local) as clocks:
        barrier()
        ev0.record(stream)
        for _ in range(args.steps):
            step(*ptrs)
        ev1.record(stream)
        barrier()
    C.check(C.lib().spattn_profile_enable(0))
    launches = (C.lib().spattn_launch_count() - n0) / args.steps
    step_bytes = 0  # send-side bytes per rank per step (all_to_all + p2p + ...), library counters
    for prim in range(len(C.PRIMITIVES)):
        calls_, bytes_ = ctypes.c_int64(), ctypes.c_int64()
        C.check(C.lib().spattn_ctx_stats(ctx, prim, ctypes.byref(calls_), ctypes.byref(bytes_)))
        step_bytes += bytes_.value
    step_bytes /= args.steps
    ms = max_over_ranks(ev0.elapsed_time(ev1)) / args.steps
    kms, kn = (ctypes.c_double * 2)(), (ctypes.c_int64 * 2)()
    C.check(C.lib().spattn_profile_read(kms, kn))
    tokens_per_s = L / (ms / 1000.0)

    # e2e through the C-ABI with HOST buffers (spattn_step_host): the H2D of q, k, v, dout
    # from pinned memory, fwd + bwd, and the D2H of dq, dk, dv (the step's result) are all
    # inside the timed region; the library pipelines the copies against the kernels over
    # kv-head groups
    def measure_e2e():
        hq, hk, hv, hdo = (x.cpu().pin_memory() for x in (q, k, v, do))
        hdq, hdk, hdv = (torch.empty_like(x, device="cpu").pin_memory() for x in (dq, dk, dv))

        def host_step():
            C.check(C.lib().spattn_step_host(
                ctx, eid, ctypes.byref(cfg), ctypes.byref(lay), 1, hq.data_ptr(), hk.data_ptr(),
                hv.data_ptr(), hdo.data_ptr(), None, None, hdq.data_ptr(), hdk.data_ptr(),
                hdv.data_ptr(), None, 0, args.e2e_groups))

        for _ in range(2):
            host_step()
        barrier()
        ev0.record(stream)
        for _ in range(args.steps):
            host_step()
        ev1.record(stream)
        barrier()
        ems = max_over_ranks(ev0.elapsed_time(ev1)) / args.steps
        h2d = sum(x.numel() * x.element_size() for x in (hq, hk, hv, hdo))
        d2h = sum(x.numel() * x.element_size() for x in (hdq, hdk, hdv))
        groups = args.e2e_groups or C.lib().spattn_pick_step_groups_len(eid, ctypes.byref(cfg), sp, lloc)
        return {"value": L / (ems / 1000.0), "unit": "tokens/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "ms_per_step": ems,
                "api": "spattn_step_host (C ABI, pinned host buffers)", "head_groups": groups}

    def secondary(name, sh, sk, sd, sL, seng):
        """The same device-timed fwd+bwd step for another workload on this context (fewer
        steps): tokens/s and the attention kernels' TFLOP/s."""
        smode = "zigzag" if seng == "ring" else "naive"
        slay = C.make_layout(smode, sL, sp)
        scfg = C.make_config(sh, sk, sd, True)
        sl = sL // sp
        mk2 = lambda h: torch.randn(1, sl, h, sd, device="cuda", dtype=torch.bfloat16, generator=g)  # noqa
        t = [mk2(sh), mk2(sk), mk2(sk), mk2(sh)]
        o2, q2g, k2g, v2g = (torch.empty_like(x) for x in (t[0], t[0], t[1], t[2]))
        l2 = torch.empty(1, sl, sh, device="cuda", dtype=torch.float32)
        sid = C.engine_id(seng)

        def st():
            saved = ctypes.c_void_p()
            C.check(C.lib().spattn_fwd(ctx, sid, ctypes.byref(scfg), ctypes.byref(slay), 1, t[0].data_ptr(),
                                       t[1].data_ptr(), t[2].data_ptr(), o2.data_ptr(), l2.data_ptr(), None,
                                       0, ctypes.byref(saved)))
            C.check(C.lib().spattn_bwd(ctx, saved, t[3].data_ptr(), q2g.data_ptr(), k2g.data_ptr(),
                                       v2g.data_ptr()))
            C.lib().spattn_saved_free(saved)

        n = max(3, min(args.steps, 5))
        for _ in range(max(3, min(args.warmup, 3))):
            st()
        barrier()
        ev0.record(stream)
        for _ in range(n):
            st()
        ev1.record(stream)
        barrier()
        sms = max_over_ranks(ev0.elapsed_time(ev1)) / n
        del t, o2, q2g, k2g, v2g, l2
        torch.cuda.empty_cache()
        return {"workload": f"{name}: {sh}q/{sk}kv heads d={sd} seq {sL} causal bs 1", "engine": seng,
                "parallelism": f"sp{sp}", "value": sL / (sms / 1e3), "unit": "tokens/s", "ms_per_step": sms,
                "steps": n, "layer_tflops": 14 * sd * causal_pairs(sL) * sh / (sms / 1e3) / 1e12}

    sec = []
    if not args.no_secondary and args.seq_len is None:
        try:
            if args.config == "c4" and engine == "ring":
                sec.append(secondary("c4/ulysses", heads, kv, d, L, "ulysses"))
            if args.config != "c2":
                h2, k2, d2, L2, e2 = CONFIGS["c2"]
                sec.append(secondary("c2", h2, k2, d2, L2, e2))
        except Exception as ex:  # noqa: BLE001
            sec.append({"error": str(ex)[:200]})

    # the metric's second half at N>1: all-to-all NVLink GB/s of this library's collective
    # (one q-shaped sequence->head exchange, send-side bytes per rank / device time, max over ranks)
    comm = None
    if world > 1:
        try:
            a2a_out = torch.empty(1, lloc * world, heads // world, d, device="cuda", dtype=torch.bfloat16)

            def a2a():
                C.check(C.lib().spattn_all_to_all(ctx, q.data_ptr(), a2a_out.data_ptr(), 1, lloc, heads, d, 2,
                                                  2, 1))

            for _ in range(3):
                a2a()
            barrier()
            ev0.record(stream)
            for _ in range(10):
                a2a()
            ev1.record(stream)
            barrier()
            cms = max_over_ranks(ev0.elapsed_time(ev1)) / 10
            sent = q.numel() * 2 * (world - 1) / world
            comm = {"a2a_bytes_per_rank": sent, "a2a_ms": cms, "a2a_gbs": sent / (cms / 1e3) / 1e9,
                    "step_bytes_per_rank": step_bytes}
        except Exception as ex:  # noqa: BLE001
            comm = {"error": str(ex)[:200]}

    e2e = None
    if not args.no_e2e:
        try:
            e2e = measure_e2e()
        except Exception as ex:  # noqa: BLE001 - keep the device measurement if the host path fails
            print(f"bench: e2e measurement failed: {ex}", file=sys.stderr)
            e2e = {"value": None, "unit": "tokens/s", "error": str(ex)[:200]}

    burst, sustained, hbm, src = peaks()
    # algorithmic flops of this rank's attention kernels per step (reference counters:
    # 4d fwd + 10d bwd per admitted pair, attention.cpp:113, :215)
    heads_local = heads // sp if engine in ("ulysses", "dummy_head") else heads
    pairs = causal_pairs(L) * heads_local if engine != "ring" else causal_pairs(L) * heads / sp
    fwd_ms, bwd_ms = kms[0] / args.steps, kms[1] / args.steps
    kernels = {
        "attn_fwd": {"ms": fwd_ms, "tflops": 4 * d * pairs / (fwd_ms / 1e3) / 1e12 if fwd_ms else None,
                     "launch_groups_per_step": kn[0] / args.steps},
        "attn_bwd": {"ms": bwd_ms, "tflops": 10 * d * pairs / (bwd_ms / 1e3) / 1e12 if bwd_ms else None,
                     "launch_groups_per_step": kn[1] / args.steps},
    }
    dom = "attn_bwd" if bwd_ms >= fwd_ms else "attn_fwd"
    achieved = kernels[dom]["tflops"]
    traffic = None
    prof = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(prof):
        try:
            traffic = json.load(open(prof)).get(f"{args.config}/{args.family}/{dom}")
        except Exception:
            traffic = None
    roofline = {"bound": "tensor", "kernel": dom, "achieved": achieved, "peak": sustained,
                "unit": "TFLOP/s", "frac": achieved / sustained if achieved else None,
                "traffic": traffic,
                "peak_note": f"bf16 dense, {src} sustained (kernel timed inside a long step); "
                             f"burst {burst}"}
    total_flops = 14 * d * causal_pairs(L) * heads
    layer_tflops = total_flops / (ms / 1e3) / 1e12
    if rank != 0:
        torch.cuda.synchronize()
        keep._fin()  # every rank releases its communicators while CUDA is still up
        if dist:
            dist.destroy_process_group()
        return
    line = {
        "metric": METRIC, "value": tokens_per_s, "unit": "tokens/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (torch.randn bf16, seeded)",
        "config": {"workload": f"{args.config}: {MODEL_OF[args.config]} attention {heads}q/{kv}kv heads "
                               f"d={d} seq {L} causal bs 1", "engine": engine,
                   "parallelism": f"sp{world}", "global_batch": 1, "seq_len": L,
                   "kernel_family": args.family,
                   "l2": "inputs exceed L2 (q alone is %d MiB)" % (q.numel() * 2 >> 20)},
        "layer_tflops": layer_tflops,
        "roofline": roofline, "kernels": kernels,
        "gpu_launches": launches,
        "clocks": clocks.summary(),
    }
    if sec:
        line["secondary"] = sec
    if e2e:
        line["e2e"] = e2e
    if comm:
        line["comm"] = comm
    if world == 1 and not args.no_cpu_baseline:
        try:
            cb = cpu_reference_sample(heads, kv, d, L, engine=engine)
            line["cpu_baseline"] = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample",
                                                       "extrapolated")}
        except Exception as ex:  # noqa: BLE001
            line["cpu_baseline"] = {"value": None, "error": str(ex)}
    print(json.dumps(line), flush=True)
    torch.cuda.synchronize()
    keep._fin()  # release the library's streams/communicators while CUDA is still up
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
