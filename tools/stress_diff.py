"""Diff the GPU fusion against the oracle on the stress goldens (debug helper).

    DIVAS_LIB=... python tools/stress_diff.py [case ...]
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import oracle
    from tests import golden_io
    from tests.test_gpu_stress import _gpu
    names = sys.argv[1:]
    for case in golden_io.stress_cases():
        if names and case.name not in names:
            continue
        got, fb = _gpu(case)
        ref = oracle.fuse_packed(case.g, case.origin, case.dx, case.density, case.packed, case.pv,
                                 case.bc, case.bh, case.unb, early_out=False)
        bad = np.flatnonzero((got["probs"] != case.p) | (got["n_thick"] != ref["n_thick"]) |
                             (got["n_thin"] != ref["n_thin"]))
        print(case.name, "lib", os.environ.get("DIVAS_LIB", "in-tree"), "bad voxels", bad.size,
              "fallbacks", fb.cpu().tolist())
        for v in bad[:10]:
            print("  vox", v, np.unravel_index(v, (case.g,) * 3), "p", got["probs"][v], case.p[v],
                  "thick", got["n_thick"][v], ref["n_thick"][v], "thin", got["n_thin"][v],
                  ref["n_thin"][v], "rho", case.density.reshape(-1)[v], "sums", got["sw"][v], ref["sw"][v], got["st"][v], ref["st"][v])


if __name__ == "__main__":
    main()
