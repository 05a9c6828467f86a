"""CPU ORACLE — test infrastructure only.

Plain, slow, obviously-correct implementation of what the B200 path computes,
written from PAPER.md (arXiv 1501.02237, Chen & Mehta).  Only `tests/`,
`__graft_entry__.smoke()` and `bench.py` (its `cpu_baseline` leg and
`--impl reference`) may import, call, link or execute anything in this
package.  The product path (`paper_1501_02237_b200/`) never imports it and
shares no code with it; the only common module is `workloads/` (seeded input
generators, no method arithmetic).

Modules:
  snf          Smith Normal Form by Bezout row/column steps.
  binomial     Props 1-2: rank, components, P0, consistency.
  points       Prop 4: the point configuration S u {0}.
  subdivision  Regular subdivision by lifting, lower-face test;
               brute force over all (d+1)-subsets, Fractions.
  volume       Independent normalised volume by a pulling triangulation
               (no lifting) for tiny inputs.
  native       ctypes wrapper of oracle/c/bdeg_oracle.c — the same brute
               force (Cramer's rule in checked __int128) for sizes the
               Python version cannot reach in seconds.

Every function cites the passage it follows.  "parity unpinned" notes are
repeated in DESIGN.md.
"""
from .snf import smith_normal_form, det_fraction, rank_fraction  # noqa: F401
from .binomial import analyze  # noqa: F401
from .points import point_configuration  # noqa: F401
from .subdivision import (  # noqa: F401
    binom, colex_rank, colex_unrank, enumerate_lifted, degree, cell_list,
)
from .volume import nvol_pulling  # noqa: F401
