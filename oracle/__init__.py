"""CPU oracle for the HASF path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and the
--impl reference arm) may import this package.  It restates the reference
algorithm (toposmooth, /root/reference/pkg/src/toposmooth) in plain C
(hasf_oracle.c) plus small numpy helpers, and is pinned against golden vectors
produced by the imported reference (tests/golden/).
"""

from .oracle import *  # noqa: F401,F403
