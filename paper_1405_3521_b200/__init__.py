"""B200-native semi-Lagrangian HJB value iteration with independent sub-domains
(arxiv 1405.3521).  The compute lives in libhj.so (include/hj.h); see DESIGN.md."""
from . import hj  # noqa: F401
