"""The warp-sorted kernel with G warps per window (G = 1, 2, 4) against the oracle.

With G > 1 one warp of a window's group sorts x and another y, the points split into G ranges (phase A's warp
queue and phase B per range), and the G partial int64 sums meet behind the group's named barrier.  The host
takes G by batch size; ISYCOS_WS_GROUP forces it (read when the engine is created, so one process per G).
Per-point eps, n_x, n_y and the records must be bit-identical to the oracle for every G: E = 2, 4, 8 (windows
33..256 with ISYCOS_WSORTED_MIN_W = 33), ragged window counts (the last CTA's groups partly empty), ties,
duplicates, k = 1, 4, 8, KSG-1 and KSG-2.
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
st = datagen.Stream(11, 5)
n = 6000
xs = {"gauss": (datagen.f32(st.normal(n)), datagen.f32(st.normal(n))),
      "int": (np.floor(st.uniform(n) * 7).astype(np.float32), np.floor(st.uniform(n) * 7).astype(np.float32)),
      "dup": (np.repeat(datagen.f32(st.normal(n // 4)), 4)[:n], np.repeat(datagen.f32(st.normal(n // 4)), 4)[:n])}
rng = np.random.default_rng(5)
# >= 592 windows per class (not latency mode); 601 / 613 / 597: ragged last CTAs for G = 1, 2, 4
W = []
for w, cnt in ((33, 601), (47, 300), (64, 313), (65, 597), (97, 200), (128, 420), (129, 613), (200, 50), (256, 560)):
    t0 = rng.integers(0, n - w, cnt)
    W += [(int(a), int(a) + w) for a in t0]
W = np.array(W, np.int64)
# The oracle's expected values depend on the inputs only, not on G: the first process computes them (oracle/ only)
# and stores them beside the test's temporary files; the processes of the other G values load them.
import os
cache = sys.argv[2]
combos = [(name, k, variant) for name in xs for k in (1, 4, 8) for variant in (0, 1) if name == "gauss" or k != 8]
if os.path.exists(cache):
    refs = dict(np.load(cache))
else:
    refs = {}
    for name, k, variant in combos:
        x, y = xs[name]
        ref = oracle.mi_batch(x, y, W, k, variant=variant)
        key = f"{name}/{k}/{variant}/"
        for f in ("s_psi", "s_log", "zero_eps", "mi", "h", "nmi"):
            refs[key + f] = np.asarray(ref[f])
        pts = [oracle.window(x[a:b], y[a:b], k=k, variant=variant) for a, b in W]
        refs[key + "eps"] = np.concatenate([o.eps for o in pts])
        refs[key + "nx"] = np.concatenate([o.nx for o in pts])
        refs[key + "ny"] = np.concatenate([o.ny for o in pts])
    np.savez(cache + ".tmp.npz", **refs)
    os.replace(cache + ".tmp.npz", cache)
bad = 0
for name, k, variant in combos:
    x, y = xs[name]
    key = f"{name}/{k}/{variant}/"
    got = isy.isycos_mi_batch_ex(x, y, W, k, variant=variant, debug=True)
    for f in ("s_psi", "s_log", "zero_eps", "mi", "h", "nmi"):
        if not np.array_equal(np.asarray(got[f]), refs[key + f]):
            print("MISMATCH", name, k, variant, f); bad += 1
    for f in ("eps", "nx", "ny"):
        g, r = np.asarray(got[f]), refs[key + f]
        if not np.array_equal(g, r):
            off = 0
            for a, b in W:  # name the first window that differs
                if not np.array_equal(g[off:off + b - a], r[off:off + b - a]):
                    print("MISMATCH point", name, k, variant, f, a, b); bad += 1
                    break
                off += b - a
print("checked", bad)
sys.exit(1 if bad else 0)
"""


@pytest.fixture(scope="module")
def oracle_cache(tmp_path_factory):
    return str(tmp_path_factory.mktemp("wsgroup") / "oracle_refs.npz")


@pytest.mark.parametrize("group", ["1", "2", "4", "0"])
def test_warp_sorted_groups_bitwise(group, oracle_cache):
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    env = dict(os.environ, ISYCOS_WS_GROUP=group, ISYCOS_WSORTED_MIN_W="33")
    r = subprocess.run([sys.executable, "-c", CHECK, ROOT, oracle_cache], env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "checked 0" in r.stdout
