"""CPU oracle for the HE linear-layer hot path -- TEST INFRASTRUCTURE ONLY.

A numpy / Python-int restatement of the reference algorithm (CryptoTrain,
pkg/src/privtrain, arXiv 2409.16675), each function citing the reference
file:line it follows.  It is pinned against golden vectors produced by the
real reference (tests/golden/make_golden.py) and is used ONLY by:

  * tests/                        (parity checker),
  * __graft_entry__.smoke()       (one checked invocation),
  * bench.py's cpu_baseline leg   (the reference's CPU path, timed).

The product path (paper_2409_16675_b200/) never imports this package; it
fails loudly when its CUDA library is missing.
"""
