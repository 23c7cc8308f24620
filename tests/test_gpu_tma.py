"""The TMA bulk-copy variants give the same outputs as the 128-bit-load
passes: the per-view z / n min-max pass (refine_minmax_tma, DIVAS_TMA=1):
same keys and refined masks, on the golden scene and on planes whose size is
not a multiple of the TMA tile; the band pass (band_pass_tma,
DIVAS_BAND_TMA=1): same scan records, tile bands and refined masks, whole
planes and windows (ragged right and bottom edges)."""

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


BAND_SCRIPT = r'''
import sys, hashlib, numpy as np, torch
sys.path.insert(0, {root!r})
from paper_2601_04860_b200.fusion import FusionParams
from paper_2601_04860_b200.segmenter import ViewWindows, refine_bands_device
dev = torch.device("cuda", 0)
rng = np.random.default_rng(11)
nv, h, w = 3, 203, 332                    # w % 4 == 0, h not a multiple of 8
t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
raw = rng.random((nv, h, w), dtype=np.float32)
raw[:, :, : w // 3] = 0.0
z = rng.random((nv, h, w), dtype=np.float32) * 5 + 1
n = rng.integers(-1, 5, size=(nv, h, w)).astype(np.int32)
d = z + rng.normal(0, 0.01, size=(nv, h, w)).astype(np.float32)
outs = []
roi = ViewWindows([[8, 8, 301, 190], [0, 0, w - 1, h - 1], [16, 40, 40, 80]], dev)
from torch.profiler import ProfilerActivity, profile
names = set()
for r in (None, roi):
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        m, aux = refine_bands_device(t(raw), t(z), t(n), t(d), FusionParams(), 0.01, roi=r)
        torch.cuda.synchronize()
    names |= {{e.name for e in prof.events() if "band_pass" in e.name}}
    outs.append((m.cpu().numpy().tobytes() if m is not None else b"") +
                aux.records.cpu().numpy().tobytes() + aux.bands.cpu().numpy().tobytes())
print("DIGEST", hashlib.sha256(b"".join(outs)).hexdigest())
print("KERNELS", sorted(names))
'''


def _band_digest(tma):
    env = dict(os.environ, DIVAS_BAND_TMA="1" if tma else "0")
    r = subprocess.run([sys.executable, "-c", BAND_SCRIPT.format(root=ROOT)], env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    kern = [l for l in r.stdout.splitlines() if l.startswith("KERNELS")][0]
    assert ("band_pass_tma" in kern) == tma, kern       # the variant under test ran
    return [l for l in r.stdout.splitlines() if l.startswith("DIGEST")][0]


def test_tma_band_pass_matches_ldg():
    assert _band_digest(True) == _band_digest(False)
