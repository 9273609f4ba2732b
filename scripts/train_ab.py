"""A/B of liborbit2 builds on the training step: per-kernel-class ms per step (profiled
pass, CUDA events) at one config.  Usage: python scripts/train_ab.py C2 16 lib1.so lib2.so ..."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r'''
import json, sys
sys.path.insert(0, ROOT)
import numpy as np, torch
from paper_2505_04802_b200 import orbit2 as o2
from workloads import get_config, make_input, make_weights
w = get_config(CFG).replace(batch=BATCH)
ctx = o2.Context(o2.config_from(w, batch=BATCH, precision=o2.BF16))
ctx.train_bind()
blob = torch.from_numpy(make_weights(w)).cuda()
packed = ctx.prepare_weights(blob); ctx.train_prepare(blob)
x = torch.from_numpy(make_input(w, batch=BATCH)).cuda()
y = torch.randn(BATCH, w.K, w.scale * w.H, w.scale * w.W, device="cuda")
bufs = ctx.train_buffers()
for _ in range(3): ctx.train_step(packed, x, y, 1e-3, 1e-3, True, bufs)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5): ctx.train_step(packed, x, y, 1e-3, 1e-3, True, bufs)
e1.record(); torch.cuda.synchronize()
ctx.set_profiling(True)
for _ in range(3): ctx.train_step(packed, x, y, 1e-3, 1e-3, True, bufs)
torch.cuda.synchronize()
t = {k: v[1] / 3 for k, v in ctx.kernel_times().items()}
t["STEP"] = e0.elapsed_time(e1) / 5
print("RESULT " + json.dumps(t))
'''

def main():
    cfg, batch, libs = sys.argv[1], int(sys.argv[2]), sys.argv[3:]
    res = {}
    for lib in libs:
        env = dict(os.environ, ORBIT2_LIB=os.path.join(ROOT, "paper_2505_04802_b200", lib))
        code = CHILD.replace("ROOT", repr(ROOT)).replace("CFG", repr(cfg)).replace("BATCH", str(batch))
        p = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env, timeout=600)
        line = [l for l in p.stdout.splitlines() if l.startswith("RESULT ")]
        if not line:
            print(lib, "FAILED", p.stderr[-2000:])
            continue
        res[lib] = json.loads(line[0][7:])
    keys = sorted({k for r in res.values() for k in r}, key=lambda k: -max(r.get(k, 0) for r in res.values()))
    print(f"{cfg} B={batch} training step, ms per step")
    print("%-16s" % "class" + "".join("%22s" % l for l in res))
    for k in keys:
        print("%-16s" % k + "".join("%22.3f" % r.get(k, float("nan")) for r in res.values()))

if __name__ == "__main__":
    main()
