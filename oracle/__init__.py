"""oracle/ -- TEST INFRASTRUCTURE ONLY.

A plain, slow, obviously-correct CPU implementation of what the hot path of
arXiv 2602.11843 computes (truncated Neumann series by radix kernels).  Only
tests/, __graft_entry__.smoke() and bench.py's CPU-baseline / --impl reference
leg may import, link or run anything here.  It shares no code with the CUDA
library under paper_2602_11843_b200/, and neither imports the other.

Parity status per function:
  series_sum   (C-1, Eq. neumann)            -- pinned: closed forms, Q brute force, Table 3
  plan_apply   (C-2, Eq. generalradix)        -- pinned: exact plans == C-1, nilpotent prefix,
                                                Lemma 4 leading coefficients, mpmath circuit iteration
  kernels      (circuit -> [f]_j)             -- pinned: all-ones (Thm 1, Sec 2.3), printed spillover
  plan         (fewest-product plan search)   -- pinned: Table 2 counts, brute-force enumeration
"""
