"""Box-assisted phase A (sorted_phase_a_cols; the paper's box-assisted k-NN, made exact) against the oracle.

Throughput-form windows of at least ISYCOS_COL_MIN_W points search their k-NN over y-sorted columns of 32 x-sorted
positions instead of the outward scan.  The knob is read when the engine is created, so each setting runs in its
own process.  Per-point eps, n_x, n_y and the window records must be bit-identical to the oracle: Gaussian data,
integer ties, duplicated points, constant stretches, ragged and XL windows (rank-merged runs), k = 1, 3, 4, 8,
KSG-1 and KSG-2, and a search whose large windows take the throughput form.
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
st = datagen.Stream(21, 7)
n = 40_000
cfg3 = datagen.cfg3()
xs = {"gauss": (cfg3.series[0][900_000:940_000].copy(), cfg3.series[1][900_000:940_000].copy()),
      "int": (np.floor(st.uniform(n) * 9).astype(np.float32), np.floor(st.uniform(n) * 9).astype(np.float32)),
      "dup": (np.repeat(datagen.f32(st.normal(n // 4)), 4)[:n], np.repeat(datagen.f32(st.normal(n // 4)), 4)[:n])}
xc, yc = xs["gauss"][0].copy(), xs["gauss"][1].copy()
xc[5000:5300] = 0.5
yc[5000:5300] = -1.0
xs["const"] = (xc, yc)
W = np.array([(0, 257), (100, 1124), (4900, 5900), (3001, 7098), (10_000, 19_000), (20_000, 36_384), (7, 40)],
             np.int64)
bad = 0
for name, (x, y) in xs.items():
    for k in (1, 3, 4, 8):
        for variant in (0, 1):
            got = isy.isycos_mi_batch_ex(x, y, W, k, variant=variant, debug=True, unfused=True)
            ref = oracle.mi_batch(x, y, W, k, variant=variant)
            for f in ("s_psi", "s_log", "zero_eps", "mi", "h", "nmi"):
                if not np.array_equal(np.asarray(got[f]), ref[f]):
                    print("MISMATCH", name, k, variant, f); bad += 1
            if k in (3, 4) and variant == 0 or name == "int":
                off = 0
                for a, b in W:
                    w = b - a
                    if w <= 8192:
                        o = oracle.window(x[a:b], y[a:b], k=k, variant=variant)
                        for f, r in (("eps", o.eps), ("nx", o.nx), ("ny", o.ny)):
                            if not np.array_equal(got[f][off:off + w], r):
                                print("MISMATCH point", name, k, variant, f, a, b); bad += 1
                    else:  # XL: sampled points
                        for i in range(0, w, 997):
                            pe, pnx, pny = oracle.point(x[a:b], y[a:b], i, k=k, variant=variant)
                            if (got["eps"][off + i], got["nx"][off + i], got["ny"][off + i]) != (np.float32(pe), pnx, pny):
                                print("MISMATCH xl point", name, k, variant, a, b, i); bad += 1
                    off += w
wl = datagen.cfg2()
ser = [s[:30_000] for s in wl.series]
ores, ost = oracle.search(ser, wl.pairs, oracle.make_params(wl.search, s_max=4096))
gres, gst = isy.search_workload(wl, series=ser, s_max=4096, unfused=True)
if gres != ores:
    print("MISMATCH search"); bad += 1
print("checked", bad)
sys.exit(1 if bad else 0)
"""


@pytest.mark.parametrize("min_w", ["64", "2048"])
def test_box_assisted_phase_a_bitwise(min_w):
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    env = dict(os.environ, ISYCOS_COL_MIN_W=min_w)
    r = subprocess.run([sys.executable, "-c", CHECK, ROOT], env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, f"min_w {min_w}:\n{r.stdout[-3000:]}\n{r.stderr[-3000:]}"
    assert "checked 0" in r.stdout
