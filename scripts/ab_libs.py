"""Interleaved A/B of library builds in ONE process (same clocks, same inputs):

    python scripts/ab_libs.py "CFG[;CFG...]" libA.so libB.so[@FLAGS] [...] [--rounds R] [--fwd-only]

Every library is loaded as its own instance of the ctypes binding; the rounds alternate
A, B, A, B, ... and each round times K2 and K4 of every call with the library's CUDA-event timing
API.  Prints the median TF/s per (variant, call) and the ratio to the first variant."""
import argparse
import importlib.util
import json
import os
import statistics
import sys

ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..")
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402


def load_binding(lib_path, tag):
    os.environ["FLASHMASK_LIB"] = lib_path
    spec = importlib.util.spec_from_file_location(f"fm_{tag}", os.path.join(ROOT, "paper_2410_01359_b200", "flashmask.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("cfgs")
    ap.add_argument("libs", nargs="+")
    ap.add_argument("--rounds", type=int, default=6)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--flags", type=int, default=0)
    ap.add_argument("--fwd-only", action="store_true")
    args = ap.parse_args()
    flags = [int(p.split("@")[1]) if "@" in p else args.flags for p in args.libs]
    libs = [p.split("@")[0] for p in args.libs]
    libs = [p if os.path.isabs(p) else os.path.join(ROOT, "paper_2410_01359_b200", p) for p in libs]
    mods = [load_binding(p, i) for i, p in enumerate(libs)]
    dev = torch.device("cuda", 0)
    ref = mods[0]
    for cfg in args.cfgs.split(";"):
        calls, _, _ = bench.build_workload(cfg, 0, 1, bench.rho_gpu(ref))
        for c in calls:
            r = bench.Runner(ref, [c], dev)
            x = r.inputs[0]
            o, lse, dq, dk, dv = r.outs[0]
            res = {i: {"fwd": [], "bwd": []} for i in range(len(mods))}

            def run(i):
                m = mods[i]
                m.flashmask_fwd(x["q"], x["k"], x["v"], x["sri"], c["causal"], out=o, lse=lse, workspace=r.ws_f[0],
                                flags=flags[i])
                if not args.fwd_only:
                    m.flashmask_bwd(x["q"], x["k"], x["v"], o, x["do"], lse, x["sri"], c["causal"], dq=dq, dk=dk,
                                    dv=dv, workspace=r.ws_b[0], flags=flags[i])

            for i in range(len(mods)):
                run(i)
            torch.cuda.synchronize()
            for _ in range(args.rounds):
                for i, m in enumerate(mods):
                    m.flashmask_timing_enable(True, kernels=[m.FM_KERNEL_FWD, m.FM_KERNEL_BWD])
                    for _ in range(args.reps):
                        run(i)
                    torch.cuda.synchronize()
                    m.flashmask_timing_enable(False)
                    t = m.flashmask_timing_collect()
                    res[i]["fwd"].append(t["fwd"][0] / args.reps)
                    if not args.fwd_only:
                        res[i]["bwd"].append(t["bwd"][0] / args.reps)
            out = {"cfg": ":".join(cfg.split(":")[:3]), "mask": c.get("family", c["masks"][0].family)}
            for i, p in enumerate(args.libs):
                f = statistics.median(res[i]["fwd"])
                out[p] = {"fwd_tf": round(r.F_fwd / (f * 1e-3) / 1e12, 1)}
                if not args.fwd_only:
                    bb = statistics.median(res[i]["bwd"])
                    out[p]["bwd_tf"] = round(r.F_bwd / (bb * 1e-3) / 1e12, 1)
                if i > 0:
                    out[p]["fwd_ratio"] = round(statistics.median(res[0]["fwd"]) / f, 3)
                    if not args.fwd_only:
                        out[p]["bwd_ratio"] = round(statistics.median(res[0]["bwd"]) / bb, 3)
            print(json.dumps(out), flush=True)
            r.free()
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
