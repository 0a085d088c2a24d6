"""CPU oracle for the sparse-permanent hot path — TEST INFRASTRUCTURE ONLY.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` /
`--impl reference` legs may import, call, link or execute anything here.  The
product (`paper_1112_6072_b200/`) never imports it, and it never imports the
product: the two share no code (inputs come from `workloads/`).

Every function is a plain, slow, obviously-correct restatement of the paper
(Wang, Liang, Bai, Huo, "A load balancing strategy for parallel computation of
sparse permanents", PAPER.md), exact integer arithmetic (Python ints) for
permanents and IEEE fp64 with an explicitly ordered operation sequence for the
KKLLL estimator.  Citations are PAPER.md line numbers.

  permanent.py  Eq. (1) brute force; Ryser's inclusion-exclusion (R-NW family)
  hybrid.py     Eq. (2) expansion, Algorithm H_per, Algorithm PH Step 2 (BFS)
  frontier.py   row-frontier DP over used-column sets (independent pin tool)
  frontier.c    the same DP in C (cfrontier.py loads it): the n = 96 goldens
  stats.py      Kendall's tau with the tie correction, Eqs. (7)-(10), by definition
  kklll.py      Algorithm KKLLL with a counter-based RNG
  schedule.py   LS / LPT / estimated order
  crt.py        Chinese remaindering and the Bregman / row-sum bounds
  ryser_nw.c    Nijenhuis-Wilf Gray-code Ryser with exact multi-limb integers
                (CPU baseline and mid-size cross-check), via cryser.py

Parity status of each function is listed in DESIGN.md §3 ("oracle pins").
"""
