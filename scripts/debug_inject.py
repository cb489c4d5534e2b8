"""Reproduce oracle-mode (injected particle) renders on golden cases; used under compute-sanitizer."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import paper_2512_09664_b200 as pg  # noqa: E402

data = np.load("tests/golden/ref_cases.npz")
for name in data["names"]:
    c = {k.split("/", 1)[1]: data[k] for k in data.files if k.startswith(f"{name}/")}
    H, W = (int(x) for x in c["hw"])
    out = np.zeros((H, W), np.float32)
    pg.splat_accumulate(c["pos1"], c["i0_1"], c["sx_1"], c["sy_1"], c["rho_1"], c["mask1"],
                        int(c["side"]), out, 0, H)
    print(name, float(np.abs(out - c["raw1"]).max()), flush=True)
