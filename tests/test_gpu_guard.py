"""Out-of-bounds write check of every kernel class (compute-sanitizer is
refused on the GPU pool): the small step cases of tools/sanitize_case.py --
general and fast ns2d kernels, ns3d passes, slab emulation with the copy,
overlapped-copy and peer-memory exchanges, pencil grids with the fused,
unfused and packed transposes -- run in a
subprocess with SKG_GUARD=1, where every device allocation has 64 KB guard
zones; no guard byte may change."""
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


def test_no_guard_zone_writes():
    code = (
        "import sys; sys.path.insert(0, %r); sys.path.insert(0, %r)\n"
        "import sanitize_case as sc\n"
        "from paper_1807_01769_b200 import api\n"
        "for c in sorted(sc.CASES): sc.main(c)\n"
        "print('violations', api.guard_violations())\n"
        "assert api.guard_violations() == 0\n" % (str(ROOT), str(ROOT / "tools")))
    env = dict(os.environ, SKG_GUARD="1", SKG_XSCR="1")  # x-forward scratch slots on at every size
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                       timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    assert "violations 0" in r.stdout
