"""The device index invariants (SC_DCHECK in csrc/scmwu_kernel.cuh: ring stages, tile row
ranges inside the slot and the matrix, stage byte budgets, partial / fold / mailbox bounds)
hold on every entry point: tools/sanitize.py's cases run against libscmwu_checked.so
(-DSCMWU_CHECKED, built by build.py --checked and __graft_entry__.build()).  A failed check
traps and aborts the launch, so each case runs in its own process."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHECKED = os.path.join(ROOT, "paper_2405_09157_b200", "libscmwu_checked.so")

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("case", ["ses", "svm", "refine", "gen", "balanced", "baselines",
                                  "vworld"])
def test_device_invariants_hold(case):
    assert os.path.exists(CHECKED), "build the checked library: python build.py --checked"
    env = dict(os.environ, SCMWU_LIB=CHECKED)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sanitize.py"), case],
                       env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "SC_DCHECK" not in r.stdout + r.stderr, \
        (r.stdout[-2000:], r.stderr[-2000:])
    assert f"sanitize case {case}: ok" in r.stdout
