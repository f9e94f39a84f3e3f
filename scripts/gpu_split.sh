cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
timeout -s KILL 900 python -m pytest tests/test_gpu_lpt.py tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "split or lpt or gqa or random_config or deterministic" 2>&1 | tail -15
cat > /tmp/mqa.py <<'PY'
import os, sys
sys.path.insert(0, os.environ["GRAFT_REPO_ROOT"])
import torch, numpy as np, importlib.util
from workloads import masks as wm, tensors as wt
def load(lib, tag):
    os.environ["FLASHMASK_LIB"] = os.path.join(os.environ["GRAFT_REPO_ROOT"], "paper_2410_01359_b200", lib)
    spec = importlib.util.spec_from_file_location(f"fm_{tag}", os.path.join(os.environ["GRAFT_REPO_ROOT"], "paper_2410_01359_b200", "flashmask.py"))
    m = importlib.util.module_from_spec(spec); spec.loader.exec_module(m); return m
for N, H, Hkv in ((8192, 32, 1), (8192, 32, 4), (16384, 16, 1)):
    m = wm.causal_document(wm.sample_doc_lens(N, 5, np.random.default_rng(0), min_len=256))
    sri = torch.from_numpy(wm.stack([m])).cuda()
    x = {n: wt.make_tensor(n, 1, N, h, 128).cuda() for n, h in (("q", H), ("do", H), ("k", Hkv), ("v", Hkv))}
    for lib in ("libflashmask_head.so", "libflashmask.so"):
        fm = load(lib, lib[:-3])
        o, lse = fm.flashmask_fwd(x["q"], x["k"], x["v"], sri, True)
        for _ in range(3): fm.flashmask_bwd(x["q"], x["k"], x["v"], o, x["do"], lse, sri, True)
        torch.cuda.synchronize()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        ev[0].record()
        for _ in range(10): fm.flashmask_bwd(x["q"], x["k"], x["v"], o, x["do"], lse, sri, True)
        ev[1].record(); torch.cuda.synchronize()
        print(N, H, Hkv, lib, "bwd ms %.3f" % (ev[0].elapsed_time(ev[1]) / 10))
PY
true
