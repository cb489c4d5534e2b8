"""Reference-side integration: the maintainer's
ctypes stub and backend.py branch, taken verbatim from INTEGRATION.md, dropped
into a copy of the built reference package; the reference's own Sampler then
renders through libpivgen_b200.so (backend.py:12-23 -> _b200.splat_accumulate
-> pgb_splat_accumulate) and must match the unmodified reference."""

from __future__ import annotations

import json
import os
import re
import shutil
import subprocess
import sys

import numpy as np
import pytest

from oracle import reference
from _helpers import ROOT

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not reference.available(), reason="oracle/_ref not built")]


def _blocks():
    text = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    blocks = re.findall(r"```python\n(.*?)```", text, flags=re.S)
    stub = next(b for b in blocks if b.startswith("# pivgen/_b200.py"))
    patch = next(b for b in blocks if b.startswith("# backend.py"))
    return stub, "\n".join(l for l in patch.splitlines() if not l.startswith("#")) + "\n"


SCRIPT = r"""
import json, sys
import numpy as np
import pivgen
from pivgen import config, flowfield
from pivgen.pipeline import Sampler
pivgen.register_flow_function("itest", lambda x, y: (1.5 + 0.01 * y, -0.5 + 0.02 * x))
cfg = config.GeneratorConfig(image_height=64, image_width=80, batch_size=3, seed=21, threads=2,
                             seeding_density_range=(0.04, 0.08), diameter_range=(0.8, 3.0),
                             rho_range=(-0.3, 0.3), hide_probability=0.1,
                             noise=config.NoiseConfig(background_offset=0.05, gaussian_std=0.01),
                             flow_sources=(config.FlowSource(function="itest"),))
with Sampler(cfg) as s:
    b = s.next_batch()
np.savez(sys.argv[1], i1=np.asarray(b.images1), i2=np.asarray(b.images2))
print(json.dumps({"backend": pivgen.active_backend()}))
"""


def _run(pkg_root, out, extra_env):
    env = dict(os.environ)
    env.update(extra_env)
    env["PYTHONPATH"] = pkg_root + os.pathsep + reference.REF_DIR
    p = subprocess.run([sys.executable, "-c", SCRIPT, out], capture_output=True, text=True, env=env, timeout=600)
    assert p.returncode == 0, p.stderr[-3000:]
    return json.loads(p.stdout.strip().splitlines()[-1])["backend"], np.load(out)


def test_reference_sampler_through_the_b200_seam(tmp_path):
    from paper_2512_09664_b200.build import LIB_PATH, build

    build()
    stub, patch = _blocks()
    pkg = tmp_path / "ref"
    shutil.copytree(os.path.join(reference.REF_DIR, "pivgen"), pkg / "pivgen")
    (pkg / "pivgen" / "_b200.py").write_text(stub)
    be = (pkg / "pivgen" / "backend.py").read_text()
    line = 'if os.environ.get("PIVGEN_PURE_PYTHON") == "1":\n'
    assert line in be
    (pkg / "pivgen" / "backend.py").write_text(be.replace(line, patch))

    backend, ours = _run(str(pkg), str(tmp_path / "ours.npz"), {"PIVGEN_B200_LIB": LIB_PATH})
    assert backend == "b200"
    backend_ref, ref = _run(reference.REF_DIR, str(tmp_path / "ref.npz"), {})
    assert backend_ref == "native"
    for k in ("i1", "i2"):
        # same particles and the same noise stream (reference RNG); only the
        # splat differs: <= 1e-5
        assert float(np.abs(ours[k] - ref[k]).max()) <= 1e-5, k
