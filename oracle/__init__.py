"""TEST INFRASTRUCTURE ONLY — the CPU oracle.

Nothing under oracle/ may be imported by the product path (paper_2511_14102_b200/).  Only
tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs use it,
and only as the checker or the timed CPU baseline.

  ref.py            ctypes handle on oracle/_ref/libmoespeq_ref.so = the reference's own
                    control-plane sources compiled unmodified (see oracle/Makefile).
  control_plane.py  independent Python restatement of the reference control plane
                    (scheduler.cpp, sim.cpp, perfmodel.cpp), token-major (reference order) and
                    layer-major/causal (live-engine order); pinned against ref.py.
  model.py          numpy restatement of the MoE decode math (no reference implementation
                    exists: PAPER.md:466-474, 489-496, 564) -- "parity unpinned by the
                    reference"; pinned only by its own golden vectors.
"""
