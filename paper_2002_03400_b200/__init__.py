"""B200-native adaptive randomized butterfly construction (arXiv 2002.03400).

Drop-in for the reference's construction path: ``factorize`` / ``Factorizer``
/ ``HybridButterfly`` / ``BlackBoxOperator`` backed by hand-written sm_100a
kernels behind the C ABI in include/bfly_b200.h.
"""
from .api import *  # noqa: F401,F403
from .api import __all__  # noqa: F401
from . import configs  # noqa: F401
