"""FlashMask hot-path benchmark (one JSON line on rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C3] [--impl flashmask|reference]

A step = one pass of the whole hot path over one batch: K1 classification + forward
(K1, K2) + backward (K1, K3, K4, K5) through the C ABI, for every call of the workload.
Metric (BASELINE.json): effective fwd+bwd TFLOP/s with skipped tiles excluded — FLOPs =
3.5 x 4 d x (non-SKIP 128x128 tiles) x 128^2 per (batch, head) (R15), the SKIP
count coming from the library's own K1 classification.  Multi-GPU: one process per GPU
(torchrun), batch entries sharded across ranks (weak scaling) for C2/C3/C5, heads sharded
for C4 (strong scaling); NCCL only reduces the per-rank timings.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from workloads import masks as wm  # noqa: E402
from workloads import tensors as wt  # noqa: E402

PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
FALLBACK_PEAKS = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}


# ----------------------------------------------------------------------------- workloads
def _seed(*xs):
    h = 1469598103934665603
    for x in xs:
        h = ((h ^ (int(x) & 0xFFFFFFFF)) * 1099511628211) & 0xFFFFFFFFFFFF
    return h


def rho_gpu(fm):
    """Rule-R block sparsity at 128x128 from the library's K1 (product path)."""
    def f(m: wm.MaskInput) -> float:
        sri = torch.from_numpy(wm.stack([m])).cuda()
        _, _, counts = fm.flashmask_classify(sri, m.causal, class_map=False)
        c = counts[0, 0].tolist()
        return c[0] / float(sum(c))
    return f


def rho_oracle(m: wm.MaskInput) -> float:
    """Same quantity from the oracle (used only by the --impl reference arm)."""
    from oracle import flashmask_oracle as fo
    _, c, _ = fo.classify(fo.expand(m.sri, m.causal, m.N), 128, 128)
    return fo.block_sparsity(c)


def causal_doc_as_bidirectional(m: wm.MaskInput) -> wm.MaskInput:
    """Causal document mask written in the bidirectional C=2 layout (LTS, UTE = y): the upper
    interval [0, y) is exactly the causal triangle, so it batches with document masks."""
    y = np.arange(m.N)
    return wm.MaskInput(N=m.N, causal=False, C=2, sri=np.stack([m.sri[:, 0], y], 1), family=m.family + "(bidir)",
                        params=m.params)


def sft_mask_in_bucket(N, lo, hi, gidx, rho_fn, base=0, max_tries=4000):
    """SFT-style packed documents (App. A.2.1, A.4.1 P:559-561) with rule-R sparsity in
    [lo, hi): document masks (n in [2,10]) below 0.5, causal-document (n in [2,20]) above."""
    for t in range(max_tries):
        rng = np.random.default_rng(_seed(base, gidx, t, int(lo * 100)))
        if hi <= 0.5:
            lens = wm.sample_doc_lens(N, int(rng.integers(2, 11)), rng, min_len=128)
            if lo < 0.15:  # the rare low-sparsity bucket: one dominant document (SURVEY d.2)
                big = int(N * rng.uniform(0.93, 0.99))
                lens = [big, N - big]
            m = wm.document(lens)
        else:
            m = wm.causal_document(wm.sample_doc_lens(N, int(rng.integers(2, 21)), rng, min_len=128))
        rho = rho_fn(m)
        if lo <= rho < hi:
            return m if not m.causal else causal_doc_as_bidirectional(m)
    raise RuntimeError(f"no mask found in bucket [{lo},{hi})")


def build_workload(cfg: str, rank: int, world: int, rho_fn, base=0):
    """Returns (calls, config_dict, scaling).  A call = dict(masks, causal, B, N, H, d, heads, batch_ids)."""
    if cfg == "C3":
        N, H, d, B = 32768, 32, 128, 4
        buckets = [(0.1, 0.2), (0.3, 0.4), (0.55, 0.65), (0.8, 0.9)]
        gids = [rank * B + i for i in range(B)]
        masks = [sft_mask_in_bucket(N, *buckets[i], gids[i], rho_fn, base) for i in range(B)]
        calls = [dict(masks=masks, causal=False, B=B, N=N, H=H, d=d, heads=range(H), batch_ids=gids)]
        conf = {"workload": "C3: SFT-style packed documents, B=4 per GPU (one mask per sparsity bucket "
                            "10-20/30-40/55-65/80-90%), H=32, N=32768, d=128, bf16 in/out",
                "global_batch": B * world, "seq_len": N, "heads": H, "head_dim": d,
                "parallelism": f"batch-sharded x{world}", "l2": "inputs (1 GiB/tensor/GPU) larger than L2"}
        return calls, conf, "weak"
    if cfg == "C2":
        N, H, d = 8192, 32, 128
        calls = []
        rng = np.random.default_rng(_seed(base, rank, 2))
        lens = wm.sample_doc_lens(N, int(rng.integers(3, 8)), rng, min_len=128)
        docs = []
        for L in lens:
            k = int(rng.integers(2, 7))
            ans = [max(1, int(rng.uniform(0.08, 0.16) * L)) for _ in range(k)]
            docs.append((L - sum(ans), ans))
        for m in (wm.causal_document(lens), wm.share_question(docs), wm.sliding_window(N, N // 16)):
            calls.append(dict(masks=[m], causal=True, B=1, N=N, H=H, d=d, heads=range(H), batch_ids=[rank]))
        conf = {"workload": "C2: B=1 per GPU, H=32, N=8192, d=128, bf16; one call each of causal-document, "
                            "share-question and sliding-window (w=N/16) masks",
                "global_batch": world, "seq_len": N, "heads": H, "head_dim": d,
                "parallelism": f"batch-sharded x{world}", "l2": "no flush; 64 MiB/tensor (Q,K,V,dO 256 MiB) > L2"}
        return calls, conf, "weak"
    if cfg == "C4":
        N, H, d = 131072, 64, 128
        assert H % world == 0
        hs = range(rank * H // world, (rank + 1) * H // world)
        calls = []
        for k_ans in (2, 6):   # DPO, RM (App. A.2.1)
            rng = np.random.default_rng(_seed(base, k_ans, 4))
            m = wm.sample_share_question(N, int(rng.integers(11, 16)), rng, k_range=(k_ans, k_ans), min_len=512)
            calls.append(dict(masks=[m], causal=True, B=1, N=N, H=H, d=d, heads=hs, batch_ids=[0]))
        conf = {"workload": "C4: DPO (k=2) and RM (k=6) share-question masks, B=1, H=64, N=131072, d=128, bf16",
                "global_batch": 1, "seq_len": N, "heads": H, "head_dim": d,
                "parallelism": f"head-sharded x{world}", "l2": "inputs larger than L2"}
        return calls, conf, "strong"
    if cfg.startswith("C5"):
        # C5:<N>:<d>  kernel sweep of every Figure-1 family, 128K tokens, hidden 4096 (App. A.5.2)
        _, N, d = cfg.split(":") if ":" in cfg else ("C5", "8192", "128")
        N, d = int(N), int(d)
        B, H = 131072 // N, 4096 // d
        doc_rng = {8192: (3, 7), 32768: (10, 14), 131072: (11, 15)}.get(N, (3, 7))
        calls = []
        for fam in wm.FAMILIES:
            ms = [wm.sample_family(fam, N, np.random.default_rng(_seed(base, rank * B + b, len(fam))), doc_rng)
                  for b in range(B)]
            calls.append(dict(masks=ms, causal=ms[0].causal, B=B, N=N, H=H, d=d, heads=range(H),
                              batch_ids=[rank * B + b for b in range(B)], family=fam))
        conf = {"workload": f"C5: all Figure-1 families, N={N}, d={d}, B={B}, H={H} per GPU, bf16",
                "global_batch": B * world, "seq_len": N, "heads": H, "head_dim": d,
                "parallelism": f"batch-sharded x{world}", "l2": "inputs larger than L2"}
        return calls, conf, "weak"
    raise SystemExit(f"unknown config {cfg}")


# ----------------------------------------------------------------------------- helpers
def make_inputs(call, device, base=0):
    B, N, d = call["B"], call["N"], call["d"]
    nh = len(call["heads"])
    out = {}
    for name in ("q", "k", "v", "do"):
        g = torch.Generator(device=device)
        g.manual_seed(_seed(base, wt.TENSOR_IDS[name], call["batch_ids"][0], call["heads"][0], N))
        out[name] = torch.randn(B, N, nh, d, generator=g, device=device, dtype=torch.float32).to(torch.bfloat16)
    out["sri"] = torch.from_numpy(wm.stack(call["masks"], 1)).to(device)
    return out


def effective_flops(call, fm):
    """(fwd, bwd) effective FLOPs of one call from the library's K1 counts at 128x128."""
    N, d, nh = call["N"], call["d"], len(call["heads"])
    sri = torch.from_numpy(wm.stack(call["masks"], 1)).cuda()
    _, _, counts = fm.flashmask_classify(sri, call["causal"], class_map=False)
    c = counts.cpu().numpy().reshape(-1, 3)
    assert N % 128 == 0
    nonskip = float((c[:, 1] + c[:, 2]).sum())
    rho = [float(x[0]) / float(x.sum()) for x in c]
    fwd = 4.0 * d * nonskip * 128 * 128 * nh
    return fwd, 2.5 * fwd, rho


def reduce_max_over_ranks(x: float, dist=None, device="cpu") -> float:
    """Max of a per-rank scalar (timings are reported as the slowest rank).  NCCL on the GPU
    path, gloo in the CPU tests; the only collective bench.py issues besides barriers."""
    if dist is None or not dist.is_initialized():
        return x
    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.path = None

    def start(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if not self.proc:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        rows = []
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 8:
                rows.append(parts)
        os.unlink(self.path)
        if not rows:
            return None
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[4 + i].lower() == "active"})
        busy = [s for s in sm if s > 0.5 * (max(mx) if mx else 1)] or sm
        return {"sm_mhz": statistics.median(busy) if busy else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


def load_peaks():
    if os.path.exists(PEAKS_PATH):
        return json.load(open(PEAKS_PATH)), "measured"
    return dict(FALLBACK_PEAKS), "fallback"


# ----------------------------------------------------------------------------- CPU oracle
def oracle_sample_rate(call, budget_s, base=0, rows_per_block=128):
    """Time the fp64 oracle (forward rows + backward rows) on whole 128-row tiles of one
    (batch, head) of ``call`` until ``budget_s`` elapses.  Returns (effective TFLOP/s, info)."""
    from oracle import flashmask_oracle as fo
    try:
        from threadpoolctl import threadpool_info
        cores = max([i.get("num_threads", 1) for i in threadpool_info()] + [1])
    except Exception:
        cores = os.cpu_count() or 1
    m = call["masks"][0]
    N, d = call["N"], call["d"]
    g = torch.Generator()
    tens = {}
    for name in ("q", "k", "v", "do"):
        g.manual_seed(_seed(base, wt.TENSOR_IDS[name], 7, 0, N))
        tens[name] = torch.randn(N, d, generator=g).to(torch.bfloat16).double().numpy()
    vec = fo.expand(m.sri, m.causal, N)
    cm, _, _ = fo.classify(vec, 128, 128)
    T = cm.shape[0]
    order = [int(x) for x in np.random.default_rng(0).permutation(T)]
    t0 = time.perf_counter()
    flops = 0.0
    tiles = 0
    for i in order:
        rows = np.arange(i * 128, min((i + 1) * 128, N))
        fo.forward(tens["q"], tens["k"], tens["v"], vec, rows=rows)
        fo.backward_rows(tens["q"], tens["k"], tens["v"], tens["do"], vec, rows)
        flops += 3.5 * 4.0 * d * 128 * 128 * float((cm[i] != fo.SKIP).sum())
        tiles += 1
        if time.perf_counter() - t0 >= budget_s:
            break
    dt = time.perf_counter() - t0
    return flops / dt / 1e12, {"cores": cores, "seconds": dt, "row_tiles": tiles,
                               "sample": f"fp64 NumPy oracle, forward + backward of {tiles} random 128-row tiles "
                                         f"of one (batch, head) of the {m.family} mask, N={N}, d={d}"}


# ----------------------------------------------------------------------------- main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C3")
    ap.add_argument("--impl", default="flashmask", choices=["flashmask", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=12.0)
    ap.add_argument("--time-kernels", default="main", choices=["main", "all"],
                    help="kernels bracketed by CUDA events inside the timed region: main = K2 and K4 only "
                         "(events between kernels remove programmatic-dependent-launch overlap), all = every kernel")
    args = ap.parse_args()

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    assert world == args.gpus or world == 1, "launch with torchrun --nproc-per-node N for --gpus N"

    if args.impl == "reference":
        return run_reference(args, rank, world)

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)

    from paper_2410_01359_b200 import flashmask as fm

    calls, conf, scaling = build_workload(args.config, rank, world, rho_gpu(fm))
    inputs = [make_inputs(c, dev) for c in calls]
    fl = [effective_flops(c, fm) for c in calls]
    F_fwd = sum(f[0] for f in fl)
    F_bwd = sum(f[1] for f in fl)
    rhos = [r for f in fl for r in f[2]]
    ws_f = [None] * len(calls)
    ws_b = [None] * len(calls)
    outs = [None] * len(calls)

    def step():
        for ci, (c, x) in enumerate(zip(calls, inputs)):
            if ws_f[ci] is None:
                p = fm.make_params(c["B"], c["N"], len(c["heads"]), c["d"], x["sri"], c["causal"])
                ws_f[ci] = torch.empty(fm.flashmask_workspace_size(p, fm.FM_PASS_FWD), dtype=torch.uint8, device=dev)
                ws_b[ci] = torch.empty(fm.flashmask_workspace_size(p, fm.FM_PASS_BWD), dtype=torch.uint8, device=dev)
                o = torch.empty_like(x["q"])
                lse = torch.empty(c["B"], len(c["heads"]), c["N"], dtype=torch.float32, device=dev)
                outs[ci] = (o, lse, torch.empty_like(x["q"]), torch.empty_like(x["q"]), torch.empty_like(x["q"]))
            o, lse, dq, dk, dv = outs[ci]
            fm.flashmask_fwd(x["q"], x["k"], x["v"], x["sri"], c["causal"], out=o, lse=lse, workspace=ws_f[ci])
            fm.flashmask_bwd(x["q"], x["k"], x["v"], o, x["do"], lse, x["sri"], c["causal"], dq=dq, dk=dk, dv=dv,
                             workspace=ws_b[ci])

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x):
        return reduce_max_over_ranks(x, dist, dev)

    for _ in range(args.warmup):
        step()
    barrier()

    # ---------------- device-timed region ----------------
    clocks = ClockSampler(local)
    clocks.start()
    stream = torch.cuda.current_stream()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    main_kernels = [fm.FM_KERNEL_FWD, fm.FM_KERNEL_BWD]
    fm.flashmask_timing_enable(True, kernels=None if args.time_kernels == "all" else main_kernels)
    barrier()
    ev0.record(stream)
    for _ in range(args.steps):
        step()
    ev1.record(stream)
    torch.cuda.synchronize()
    fm.flashmask_timing_enable(False)
    ktimes = fm.flashmask_timing_collect()
    barrier()
    clk = clocks.stop()
    ms_total = ev0.elapsed_time(ev1)
    ms_step = max_over_ranks(ms_total / args.steps)
    # kernel split of the small kernels (K1, K3, K5) and the launch count: one extra untimed-for-
    # value step with every kernel bracketed
    fm.flashmask_timing_enable(True)
    step()
    torch.cuda.synchronize()
    fm.flashmask_timing_enable(False)
    ksplit = fm.flashmask_timing_collect()
    launches_per_step = int(sum(n for _, n in ksplit.values()))

    # ---------------- end-to-end through host buffers ----------------
    e2e = None
    if not args.no_e2e:
        # End to end through the public API from pinned host buffers: every step copies the
        # inputs in and dq/dk/dv out.  The step is split into one call per (batch entry, group of
        # HG heads) — attention heads are independent — so the copies of chunk c+1 (H2D) and c-1
        # (D2H) overlap the kernels of chunk c on 3 streams and pipeline fill/drain is short.  The
        # host buffers hold each chunk contiguously ([1, N, HG, d]), chosen at setup.
        chunks = []
        for ci, (c, x) in enumerate(zip(calls, inputs)):
            H = len(c["heads"])
            HG = int(os.environ.get("FM_E2E_HEADS", "8"))
            HG = HG if H % HG == 0 else H
            for bi in range(c["B"]):
                for h0 in range(0, H, HG):
                    hx = {k: (v[bi:bi + 1, :, h0:h0 + HG] if k != "sri" else v[bi:bi + 1]).contiguous().cpu()
                          .pin_memory() for k, v in x.items()}
                    dx = {k: torch.empty(t.shape, dtype=t.dtype, device=dev) for k, t in hx.items()}
                    do_ = (torch.empty_like(dx["q"]), torch.empty(1, HG, c["N"], dtype=torch.float32, device=dev),
                           torch.empty_like(dx["q"]), torch.empty_like(dx["k"]), torch.empty_like(dx["v"]))
                    ho = tuple(torch.empty(t.shape, dtype=t.dtype).pin_memory() for t in do_[2:])
                    chunks.append((c, hx, dx, do_, ho))
        wsf = torch.empty(max(w.numel() for w in ws_f), dtype=torch.uint8, device=dev)
        wsb = torch.empty(max(w.numel() for w in ws_b), dtype=torch.uint8, device=dev)
        h2d = sum(t.numel() * t.element_size() for ch in chunks for t in ch[1].values())
        d2h = sum(t.numel() * t.element_size() for ch in chunks for t in ch[4])
        s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()

        # Consecutive steps pipeline like a training loop that prefetches its next batch: step
        # k+1's H2D of chunk c waits only for step k's kernels of chunk c (its device input
        # buffers), and its kernels of chunk c for step k's D2H of chunk c (its output buffers).
        done = [None] * len(chunks)  # per chunk: kernels of the last step finished
        out = [None] * len(chunks)   # per chunk: D2H of the last step finished

        def e2e_step():
            ev_in = []
            for i, (c, hx, dx, _, _) in enumerate(chunks):
                with torch.cuda.stream(s_in):
                    if done[i] is not None:
                        s_in.wait_event(done[i])
                    for k, v in hx.items():
                        dx[k].copy_(v, non_blocking=True)
                    e = torch.cuda.Event()
                    e.record(s_in)
                    ev_in.append(e)
            for i, ((c, hx, dx, do_, ho), e) in enumerate(zip(chunks, ev_in)):
                stream.wait_event(e)
                if out[i] is not None:
                    stream.wait_event(out[i])
                o, lse, dq, dk, dv = do_
                fm.flashmask_fwd(dx["q"], dx["k"], dx["v"], dx["sri"], c["causal"], out=o, lse=lse, workspace=wsf)
                fm.flashmask_bwd(dx["q"], dx["k"], dx["v"], o, dx["do"], lse, dx["sri"], c["causal"], dq=dq, dk=dk,
                                 dv=dv, workspace=wsb)
                done[i] = torch.cuda.Event()
                done[i].record(stream)
                with torch.cuda.stream(s_out):
                    s_out.wait_event(done[i])
                    for hdst, dsrc in zip(ho, (dq, dk, dv)):
                        hdst.copy_(dsrc, non_blocking=True)
                    out[i] = torch.cuda.Event()
                    out[i].record(s_out)

        def e2e_drain():  # every D2H issued so far has landed in host memory
            for ev in out:
                stream.wait_event(ev)

        e2e_step()
        e2e_drain()
        torch.cuda.synchronize()
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        s_in.wait_event(e0)
        s_out.wait_event(e0)
        n_e2e = max(1, min(args.steps, 5))
        for _ in range(n_e2e):
            e2e_step()
        e2e_drain()
        e1.record(stream)
        torch.cuda.synchronize()
        e2e_ms = max_over_ranks(e0.elapsed_time(e1) / n_e2e)
        e2e = {"value": round(world * (F_fwd + F_bwd) / (e2e_ms * 1e-3) / 1e12, 2), "unit": "TFLOP/s",
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "ms_per_step": round(e2e_ms, 3),
               "pipeline": f"one call per (batch entry, {HG}-head group), H2D / kernels / D2H on 3 streams; "
                           "host buffers chunk-contiguous; step k+1's copies overlap step k's kernels (prefetch)"}

    # ---------------- report ----------------
    value = world * (F_fwd + F_bwd) / (ms_step * 1e-3) / 1e12
    peaks, peak_src = load_peaks()
    peak_sust = peaks.get("bf16_tflops_sustained", peaks["bf16_tflops"])
    traffic = None
    tpath = os.path.join(ROOT, "profiles", f"traffic_{args.config}.json")
    if os.path.exists(tpath):
        traffic = json.load(open(tpath)).get("fm_bwd_kernel_bytes_per_launch")
    k_bwd_ms, k_bwd_n = ktimes["bwd"]
    k_fwd_ms, k_fwd_n = ktimes["fwd"]
    bwd_tf = F_bwd * args.steps / (k_bwd_ms * 1e-3) / 1e12 if k_bwd_ms > 0 else None
    fwd_tf = F_fwd * args.steps / (k_fwd_ms * 1e-3) / 1e12 if k_fwd_ms > 0 else None
    launches = launches_per_step * args.steps

    cpu = None
    if rank == 0 and world == 1:
        rate, info = oracle_sample_rate(calls[0], args.cpu_budget)
        cpu = {"value": round(rate, 6), "unit": "TFLOP/s", "cores": info["cores"], "kind": "oracle",
               "sample": info["sample"], "seconds": round(info["seconds"], 2)}

    if rank == 0:
        line = {
            "metric": "effective fwd+bwd TFLOPs/s (skipped tiles excluded) and % of B200 bf16 peak",
            "value": round(value, 2), "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms_step, 3), "higher_is_better": True,
            "scaling": scaling, "vs_baseline": None, "dtype": "bf16", "data": "synthetic (seeded N(0,1) "
            "q/k/v/dO, generated masks)", "config": conf,
            "pct_of_peak": round(100.0 * value / world / peak_sust, 2), "peak_tflops": peak_sust,
            "peak_source": f"{peak_src} bf16_tflops_sustained",
            "tokens_per_s": round(world * sum(c["B"] * c["N"] for c in calls) / (ms_step * 1e-3), 1),
            "fwd_tflops_kernel": round(fwd_tf, 2) if fwd_tf else None,
            "bwd_tflops_kernel": round(bwd_tf, 2) if bwd_tf else None,
            "block_sparsity_128": [round(r, 4) for r in rhos],
            "kernels_ms_per_step": {k: round((ktimes[k][0] / args.steps) if ktimes[k][1] else v[0], 4)
                                    for k, v in ksplit.items()},
            "kernel_timing": "fwd/bwd: CUDA events on the launch stream inside the timed region; others: one "
                             "extra step with every kernel bracketed" if args.time_kernels == "main" else
                             "every kernel bracketed inside the timed region",
            "roofline": {"kernel": "fm_bwd_kernel (K4)", "bound": "tensor",
                         "achieved": round(bwd_tf, 2) if bwd_tf else None, "peak": peak_sust, "unit": "TFLOP/s",
                         "frac": round(bwd_tf / peak_sust, 4) if bwd_tf else None, "traffic": traffic,
                         "traffic_unit": "bytes per launch (dram read+write, ncu --set full)",
                         "algorithmic": "10*128^2*d FLOPs per non-SKIP 128x128 tile (SURVEY d.5)"},
            "e2e": e2e, "gpu_launches": launches, "clocks": clk, "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


def run_reference(args, rank, world):
    """--impl reference: the fp64 oracle as it stands on the host cores, same metric/unit."""
    if rank != 0:
        return
    # same workload (same seeds) as the CUDA arm; buckets picked with the oracle's own
    # classification, which is bit-exact with K1 (tests/test_gpu_parity.py)
    calls, conf, _ = build_workload(args.config, 0, 1, rho_oracle)
    flat = [dict(c, masks=[m]) for c in calls for m in c["masks"]]
    rates = []
    info = None
    per_step = max(0.5, min(6.0, 150.0 / max(1, args.steps + args.warmup)))
    for s in range(args.warmup + args.steps):
        r, info = oracle_sample_rate(flat[s % len(flat)], per_step)
        if s >= args.warmup:
            rates.append(r)
    value = statistics.mean(rates)
    ms_step = per_step * 1e3
    line = {"impl": "reference", "metric": "effective fwd+bwd TFLOPs/s (skipped tiles excluded) and % of B200 bf16 peak",
            "value": round(value, 6), "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms_step, 1), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": conf,
            "cpu_baseline": {"value": round(value, 6), "unit": "TFLOP/s", "cores": info["cores"], "kind": "oracle",
                             "sample": info["sample"] + f"; {per_step:.1f} s per step"},
            "e2e": {"value": round(value, 6), "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
