"""Debug: run C1 through the fp32 path once and report finiteness / error vs the oracle."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from gpu_helpers import run_cuda, rel_err  # noqa: E402
from paper_2505_04802_b200 import orbit2 as o2  # noqa: E402
from workloads import get_config, make_input, make_weights  # noqa: E402

prec = int(sys.argv[1]) if len(sys.argv) > 1 else o2.FP32
w = get_config("C1")
x = make_input(w)
blob = make_weights(w)
for rep in range(3):
    got = run_cuda(w, x, blob, prec)
    print("rep", rep, "finite", np.isfinite(got).all(), "nan rows", np.where(~np.isfinite(got).all(axis=(0, 1, 3)))[0][:5])
