"""A/B timing of library builds: per-kernel-class ms of one forward (event-timed).

    python scripts/ab_kernels.py [CONFIG] [BATCH] [REPS]
Runs itself once per lib in $AB_LIBS (space-separated .so paths; default: the
in-tree liborbit2.so), each in a fresh process with ORBIT2_LIB set, and prints
a table.  Also prints the max |diff| of the output against the first lib.
"""
import json
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def child(cfg_name, batch, reps, dump):
    import torch
    sys.path.insert(0, ROOT)
    from paper_2505_04802_b200 import orbit2 as o2
    from workloads import get_config, make_input, make_weights
    w = get_config(cfg_name, batch=batch)
    ctx = o2.Context(o2.config_from(w))
    x = torch.from_numpy(make_input(w)).cuda()
    packed = ctx.prepare_weights(torch.from_numpy(make_weights(w)).cuda())
    out = ctx.forward(packed, x)
    for _ in range(2):
        ctx.forward(packed, x, out=out)
    torch.cuda.synchronize()
    ctx.set_profiling(True)
    for _ in range(reps):
        ctx.forward(packed, x, out=out)
    torch.cuda.synchronize()
    kt = ctx.kernel_times()
    ctx.set_profiling(False)
    np.save(dump, out[:, :, ::7, ::7].float().cpu().numpy())
    print(json.dumps({k: v[1] / reps for k, v in kt.items()}))


def main():
    if len(sys.argv) > 1 and sys.argv[1] == "--child":
        child(sys.argv[2], int(sys.argv[3]), int(sys.argv[4]), sys.argv[5])
        return
    cfg_name = sys.argv[1] if len(sys.argv) > 1 else "C2"
    batch = int(sys.argv[2]) if len(sys.argv) > 2 else 64
    reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
    libs = os.environ.get("AB_LIBS", os.path.join(ROOT, "paper_2505_04802_b200", "liborbit2.so")).split()
    rows, outs = [], []
    for i, lib in enumerate(libs):
        dump = f"/tmp/ab_out_{i}.npy"
        env = dict(os.environ, ORBIT2_LIB=lib)
        r = subprocess.run([sys.executable, __file__, "--child", cfg_name, str(batch), str(reps), dump],
                           env=env, capture_output=True, text=True)
        if r.returncode != 0:
            print(f"{lib}: FAILED\n{r.stderr[-2000:]}")
            continue
        rows.append((os.path.basename(lib), json.loads(r.stdout.strip().splitlines()[-1])))
        outs.append(np.load(dump))
    keys = sorted({k for _, d in rows for k in d}, key=lambda k: -rows[0][1].get(k, 0))
    print(f"{cfg_name} B={batch}, ms per forward (mean of {reps})")
    print("kernel".ljust(18) + "".join(n[:22].rjust(24) for n, _ in rows))
    for k in keys + ["TOTAL"]:
        vals = [sum(d.values()) if k == "TOTAL" else d.get(k, float("nan")) for _, d in rows]
        print(k.ljust(18) + "".join(f"{v:24.3f}" for v in vals))
    for (n, _), o in zip(rows[1:], outs[1:]):
        print(f"max|out - out[{rows[0][0]}]| for {n}: {np.abs(o - outs[0]).max():.3e}")


if __name__ == "__main__":
    main()
