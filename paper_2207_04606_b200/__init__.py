"""B200-native composable-format sparse operator path (SparseTIR / strata hot path).

See DESIGN.md.  All compute runs in libstrata_b200.so (sm_100a); importing fails loudly when
the extension has not been built.
"""
from .ops import *  # noqa: F401,F403
from .ops import __all__  # noqa: F401
