"""CPU oracle for the SCMWU hot path — TEST INFRASTRUCTURE ONLY.

This package restates, in numpy, the reference's per-iteration algorithm
(normalized spectral exponential, SES / SVM oracles, progress measures,
the feasibility-test loops and the adaptive search) so that the CUDA path can
be checked against it on the GPU box, where the reference itself is absent.

Rules:
  * only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
    --impl reference legs may import it, and only as the checker or the
    CPU baseline — never as the thing measured or shipped;
  * the product package (paper_2405_09157_b200) never imports it and has no
    CPU fallback;
  * it is pinned against golden vectors produced by the real reference
    (tests/golden/make_golden.py → tests/golden/*.json), see
    tests/test_oracle_golden.py.
"""
from .scmwu_oracle import *  # noqa: F401,F403
