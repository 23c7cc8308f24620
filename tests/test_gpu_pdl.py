"""Programmatic dependent launch (the kernel chains launched with
programmatic stream serialization, each kernel opening with
griddepcontrol.wait) changes no bit: the windowed refine + band pass and the
one-call fusion of the sphere_on_plane scene, under a CUDA graph replay as
the bench runs them, give the same records, bands, votes and probabilities
with DIVAS_PDL=1 and DIVAS_PDL=0."""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r'''
import sys, hashlib, numpy as np, torch
sys.path.insert(0, {root!r})
from tests import golden_io
from tests.gpu_cases import bounds_ns, device_views, grid_ns
from paper_2601_04860_b200.fusion import Fuser
from paper_2601_04860_b200.segmenter import refine_bands_device
dev = torch.device("cuda", 0)
case = golden_io.scene_cases()["sop"]
raw, z, _ref = golden_io.scene_raw()
t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
rr, zz, nn, dd = t(raw), t(z), t(case.nsamps), t(case.dexps)
dv = device_views(case, dev)
fuser = Fuser(grid_ns(case), case.pv, bounds_ns(case))
dens = t(case.density.reshape(-1))
outs = []
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    m, aux = refine_bands_device(rr, zz, nn, dd, case.pv, case.dx)
    out = fuser.run(dens, dv, stats=True, occ=True)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        m2, aux2 = refine_bands_device(rr, zz, nn, dd, case.pv, case.dx, aux=aux, out=m)
        out2 = fuser.run(dens, dv, stats=True, occ=True, workspace=out["workspace"])
    g.replay()
torch.cuda.synchronize()
for x in (m, aux.records, aux.bands, out2["probs"], out2["n_thick"], out2["n_thin"],
          out2["occ"]):
    outs.append(x.cpu().numpy().tobytes())
print("DIGEST", hashlib.sha256(b"".join(outs)).hexdigest())
'''


def _digest(pdl):
    env = dict(os.environ, DIVAS_PDL="1" if pdl else "0")
    r = subprocess.run([sys.executable, "-c", SCRIPT.format(root=ROOT)], env=env,
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    return [l for l in r.stdout.splitlines() if l.startswith("DIGEST")][0]


def test_pdl_changes_no_bit():
    assert _digest(True) == _digest(False)
