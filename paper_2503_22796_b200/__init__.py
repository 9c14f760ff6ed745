"""B200-native (sm_100a) drop-in for DiTFastAttnV2's fused head-wise attention
path: per-head Full / Arrow / Cached plans, the joint text+image attention
call, and the calibration RSE query. See DESIGN.md and include/dfa2c.h."""
from .api import *  # noqa: F401,F403
from . import api  # noqa: F401

__version__ = "0.1.0"
