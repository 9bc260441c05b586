"""a4's warp-ballot count form (north star; SURVEY §8(a) a4 option 1) against the oracle.

The small-window kernel (one warp per window, w <= 256) carries both count forms: per-lane predicated adds
(default) and ballot + popc over 32 candidates for one warp-uniform point (ISYCOS_KNN_MODE bit 1).  The knob is
read when the engine is created, so each mode runs in its own process.  Both must give per-point n_x, n_y and
the window records bit-identical to the oracle (ties, duplicates, constant windows, KSG-1 and KSG-2).
"""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHECK = r"""
import sys
import numpy as np
sys.path.insert(0, sys.argv[1])
import datagen, oracle
import paper_2204_09131_b200 as isy
st = datagen.Stream(7, 3)
n = 5000
xs = {"gauss": (datagen.f32(st.normal(n)), datagen.f32(st.normal(n))),
      "int": (np.floor(st.uniform(n) * 6).astype(np.float32), np.floor(st.uniform(n) * 6).astype(np.float32)),
      "dup": (np.repeat(datagen.f32(st.normal(n // 4)), 4)[:n], np.repeat(datagen.f32(st.normal(n // 4)), 4)[:n])}
xc, yc = xs["int"][0].copy(), xs["int"][1].copy()
xc[2000:2100] = 1.0
yc[2000:2100] = 2.0
xs["const"] = (xc, yc)
# >= 592 windows per size class, so the batch runs the warp-per-window kernel (not latency mode)
W = np.array([(a, a + w) for w in (6, 17, 32, 33, 50, 64) for a in range(0, 4000, 7)] + [(2000, 2060), (1990, 2050)],
             np.int64)
bad = 0
for name, (x, y) in xs.items():
    for k in (1, 4):
        for variant in (0, 1):
            Wk = W[(W[:, 1] - W[:, 0]) > k]
            got = isy.isycos_mi_batch_ex(x, y, Wk, k, variant=variant, debug=True)
            ref = oracle.mi_batch(x, y, Wk, k, variant=variant)
            for f in ("s_psi", "s_log", "zero_eps", "mi"):
                if not np.array_equal(np.asarray(got[f]), ref[f]):
                    print("MISMATCH", name, k, variant, f); bad += 1
            off = 0
            for a, b in Wk:
                o = oracle.window(x[a:b], y[a:b], k=k, variant=variant)
                w = b - a
                for f, r in (("eps", o.eps), ("nx", o.nx), ("ny", o.ny)):
                    if not np.array_equal(got[f][off:off + w], r):
                        print("MISMATCH point", name, k, variant, f, a, b); bad += 1
                off += w
print("checked", bad)
sys.exit(1 if bad else 0)
"""


@pytest.mark.parametrize("mode", ["1", "3", "2"])  # branch-free + per-lane (default), + ballot, guarded + ballot
def test_count_forms_bitwise(mode):
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    env = dict(os.environ, ISYCOS_KNN_MODE=mode)
    r = subprocess.run([sys.executable, "-c", CHECK, ROOT], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, f"mode {mode}:\n{r.stdout[-3000:]}\n{r.stderr[-3000:]}"
    assert "checked 0" in r.stdout
