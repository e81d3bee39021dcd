"""CPU oracle for the SLAMCast hot path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs may import this package, and only as the checker
or the CPU baseline.  The product (paper_1805_03709_b200) never imports it.

Parity pinning: the restatements here are checked against golden vectors
generated from the reference implementation itself
(tests/golden/gen_golden.py imports /root/reference/pkg/src/voxelstream in
the build container) and against the reference's pipeline digest
``model_sha256`` (pkg/fixtures/protocol/manifest.json).  Quantised TSDF
bytes and the compaction format have no reference implementation; they are
defined normatively here (mc_oracle.c) and pinned by known-answer tests.
"""

from .oracle import *  # noqa: F401,F403
