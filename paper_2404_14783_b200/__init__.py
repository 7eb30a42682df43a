"""B200-native one-pass randomized quaternion low-rank approximation
(arXiv 2404.14783): the sketch / rangefinder / core-solve hot path as sm_100a
CUDA kernels behind the reference's API.  See DESIGN.md."""
from .qlra import *  # noqa: F401,F403
from . import qlra  # noqa: F401
