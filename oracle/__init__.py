"""CPU oracle for the batchsim-b200 hot path -- TEST INFRASTRUCTURE ONLY.

A from-scratch numpy restatement of the reference algorithm (pose algebra:
/root/reference/pkg/src/batchsim/pose.py; everything downstream: /root/reference/SPEC.md,
with the SPEC-silent choices fixed in DESIGN.md "Decisions register").  Every function cites
the reference line it follows.

Who may import this package: tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference legs -- as the CHECKER or the timed CPU baseline, never as product code.
The product package (paper_2410_00425_b200) never imports it; it has no CPU fallback.

Pinning: the pose algebra is pinned bit-for-bit against golden vectors generated from the
reference itself (tests/golden/make_pose_golden.py -> tests/golden/pose_golden.npz).  The
dynamics/render restatements have no reference code to run (the reference ships only
SPEC.md for them): they are pinned by the SPEC's known-answer examples (tests/test_oracle_*).
"""
