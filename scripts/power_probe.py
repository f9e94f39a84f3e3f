"""Run the forward and the backward kernel alone in a loop and sample SM clock, power and
throttle reasons meanwhile: tells whether each kernel runs power-capped (then energy per
FLOP, not cycles, bounds it)."""
import os
import subprocess
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2410_01359_b200 import flashmask as fm  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
secs = float(sys.argv[2]) if len(sys.argv) > 2 else 4.0
calls, conf, _ = bench.build_workload(cfg, 0, 1, bench.rho_gpu(fm))
c = calls[0]
dev = torch.device("cuda", 0)
x = bench.make_inputs(c, dev)
ff, fb, _ = bench.effective_flops(c, fm)[:3]
o, lse = fm.flashmask_fwd(x["q"], x["k"], x["v"], x["sri"], c["causal"])
fm.flashmask_bwd(x["q"], x["k"], x["v"], o, x["do"], lse, x["sri"], c["causal"])
torch.cuda.synchronize()


def sample(fn, flops):
    p = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw,clocks_throttle_reasons.active",
                          "--format=csv,noheader,nounits", "-lms", "100"], stdout=subprocess.PIPE, text=True)
    t0 = time.time()
    n = 0
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    while time.time() - t0 < secs:
        for _ in range(4):
            fn()
            n += 1
        torch.cuda.synchronize()
    ev1.record()
    torch.cuda.synchronize()
    p.terminate()
    out = p.communicate()[0].strip().splitlines()
    rows = [r.split(",") for r in out[len(out) // 4:]]
    mhz = sorted(float(r[0]) for r in rows)
    pw = sorted(float(r[1]) for r in rows)
    reasons = sorted(set(r[2].strip() for r in rows))
    ms = ev0.elapsed_time(ev1) / n
    return mhz[len(mhz) // 2], pw[len(pw) // 2], reasons, ms, flops / ms / 1e9


for name, fn, fl in (("fwd", lambda: fm.flashmask_fwd(x["q"], x["k"], x["v"], x["sri"], c["causal"]), ff),
                     ("bwd", lambda: fm.flashmask_bwd(x["q"], x["k"], x["v"], o, x["do"], lse, x["sri"], c["causal"]),
                      fb)):
    mhz, pw, rs, ms, tf = sample(fn, fl)
    print(f"{cfg} {name}: sm {mhz:.0f} MHz  power {pw:.0f} W  reasons {rs}  {ms:.2f} ms  {tf:.1f} TF/s "
          f"({tf / mhz:.3f} TF/s per MHz)", flush=True)
