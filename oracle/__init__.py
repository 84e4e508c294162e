"""TEST INFRASTRUCTURE ONLY — parity checkers for libswt_b200.

* ``oracle.swt_oracle`` — float64 CPU restatement of the reference path
  (C for the sequential parts, numpy for dense linear algebra).
* ``oracle.ref``        — the unmodified reference engine compiled from
  /root/reference into oracle/_ref/ (present when built in the dev container;
  the prebuilt .so travels to the GPU box).

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline / reference
arm) may import this package, and only as the checker; the product package
paper_2211_16270_b200 never does.
"""
