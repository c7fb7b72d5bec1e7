"""ORACLE — test infrastructure only.

A plain, slow, obviously-correct CPU implementation of what the hot path
computes, written from PAPER.md (Ghosh & Chaudhury, arXiv 1605.02178) in
binary64 (numpy) with the Chebyshev coefficients in extended precision
(mpmath).  Citations: `P:<line>` = /root/reference/PAPER.md line.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` /
`--impl reference` legs may import this package.  It shares no code with the
CUDA path (`paper_1605_02178_b200/`) and never imports it; the only module both
sides read is `synth/` (seeded inputs, no method arithmetic).

Modules
  chebyshev  eqs. (11)-(16), (18), (19), Taylor c_n        [pinned: tests/test_oracle_chebyshev.py]
  filters    eqs. (1), (6)-(10), (17), GCF pipeline         [pinned: tests/test_oracle_filters.py]
  deriche    the Deriche-class recursive fast mode (NEXT-1)  [pinned: tests/test_oracle_deriche.py]

Every function is pinned by at least one check that does not re-use its own
formula (closed forms, library special cases, brute force, limits); see
DESIGN.md §"Oracle pins".  No function here is "parity unpinned".
"""
from .chebyshev import (  # noqa: F401
    cheb_T,
    cheb_T_recurrence,
    cheb_c,
    cheb_c_float,
    cheb_d,
    cheb_zeros,
    monomial_table,
    mu_of,
    required_dps,
    taylor_c,
)
from .filters import (  # noqa: F401
    bilateral_direct,
    gauss_fir,
    gc_bruteforce,
    gc_filter,
    gc_filter_rows,
    max_abs,
    mirror_index,
    mse_db,
    psnr_db,
    rms,
    spatial_taps,
)
from .deriche import (  # noqa: F401
    DERICHE,
    deriche_2d,
    deriche_coeffs,
    deriche_filter_1d,
    deriche_kernel,
    deriche_pad,
    gc_filter_deriche,
)
