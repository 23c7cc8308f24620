"""The TMA bulk-copy variant of the per-view z / n min-max pass
(refine_minmax_tma, selected with DIVAS_TMA=1) gives the same keys and the
same refined masks as the 128-bit-load pass, on the golden scene and on
planes whose size is not a multiple of the TMA tile."""

import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r'''
import sys, numpy as np, torch
sys.path.insert(0, {root!r})
from tests import golden_io
from paper_2601_04860_b200.segmenter import refine_minmax_device, refine_masks_device
dev = torch.device("cuda", 0)
raw, z, _ref = golden_io.scene_raw()
case = golden_io.scene_cases()["sop"]
rng = np.random.default_rng(7)
outs = []
for (zz, nn, rr) in [(z, case.nsamps, raw),
                     (rng.random((5, 333, 1212), dtype=np.float32) * 9 + 0.5,
                      rng.integers(-1, 4, size=(5, 333, 1212)).astype(np.int32),
                      rng.random((5, 333, 1212), dtype=np.float32))]:
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    k = refine_minmax_device(t(zz), t(nn))
    m = refine_masks_device(t(rr), t(zz), t(nn))
    torch.cuda.synchronize()
    outs.append(k.cpu().numpy().tobytes() + m.cpu().numpy().tobytes())
import hashlib
print("DIGEST", hashlib.sha256(b"".join(outs)).hexdigest())
'''


def _digest(tma):
    env = dict(os.environ, DIVAS_TMA="1" if tma else "0")
    r = subprocess.run([sys.executable, "-c", SCRIPT.format(root=ROOT)], env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    return [l for l in r.stdout.splitlines() if l.startswith("DIGEST")][0]


def test_tma_minmax_matches_ldg():
    assert _digest(True) == _digest(False)
