"""T5 (SURVEY §4.2, §5 "Race detection") without compute-sanitizer, which is closed on the GPU pool
(profiles/r02_sanitizer_closed.log).  scripts/sanitize_workload.py launches every kernel family (KSG-1 and
KSG-2, brute force, latency mode, warp-sorted, fused, throughput sort + scan with the XL merge and the NEXT-3
block sort, and a pipelined search), checks each against the oracle and repeats each batch in-process.
Here it runs once plain and once per poison byte: with ISYCOS_POISON every kernel first fills its shared
memory with the byte and the engine fills the scan scratch and record buffers, so reading anything not
written in the batch, or a shared-memory read racing a write, changes the outputs.  All dumps must be
bitwise identical."""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_poisoned_runs_identical(tmp_path):
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    dumps = []
    for poison in (None, "0x00", "0xff", "0x7f", "0xa5"):
        env = dict(os.environ)
        env.pop("ISYCOS_POISON", None)
        if poison is not None:
            env["ISYCOS_POISON"] = poison
        out = tmp_path / f"dump_{poison}.npz"
        r = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "sanitize_workload.py"), "--dump", str(out),
                            "--repeat", "3"], env=env, capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, f"poison {poison}:\n{r.stdout[-3000:]}\n{r.stderr[-3000:]}"
        dumps.append(np.load(out))
    base = dumps[0]
    for d in dumps[1:]:
        assert sorted(d.files) == sorted(base.files)
        for f in base.files:
            assert np.array_equal(d[f], base[f]), f
