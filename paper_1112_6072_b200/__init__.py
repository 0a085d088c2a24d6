"""paper_1112_6072_b200 — B200-native exact sparse permanents (arXiv 1112.6072 hot path).

libsperm.so (csrc/, C ABI in include/sperm.h) holds the sm_100a kernels:
  sperm_expand    Eq. (2) BFS expansion (Algorithm PH Step 2 / H_per)
  sperm_expand_subtree  H_per below the job level, depth first in shared memory
  sperm_estimate  KKLLL approximate permanents (job weights)
  sperm_schedule  improved Step 3: non-increasing-estimate LPT
  sperm_permanent batched R-NW Gray-code leaf permanents, exact mod primes
`sperm` is the thin ctypes binding; `pipeline` sequences the calls (Algorithm PH).
"""
from .sperm import (  # noqa: F401
    KMAX, NMAX, DeviceQueue, SpermError, lib, primes, residues_to_ints, residues_to_ints_device, sperm_bound_primes, sperm_crt, sperm_estimate, sperm_estimate_stats, sperm_expand, sperm_expand_stats, sperm_expand_subtree, sperm_expand_subtree_stats, sperm_fold_mod, sperm_kendall_tau, sperm_launch_count, sperm_list_schedule, replay_efficiency, sperm_interpolate_mod, sperm_nnz, tau_z,
    sperm_permanent, sperm_permanent_host, sperm_prime, sperm_reduce_mod, sperm_rnw_stats, sperm_rnw_terms, sperm_schedule, sperm_timing_enable,
    sperm_timing_get, sperm_timing_reset, sperm_version)
