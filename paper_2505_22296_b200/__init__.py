"""B200-native sequence-parallel attention (arXiv 2505.22296 / 360-LLaMA-Factory SP layer).

Ulysses, Dummy-Head Ulysses, XTuner hidden-split (comparator), zigzag Ring and USP engines over
hand-written sm_100a kernels, behind the reference's operator API (``seqpar``) and a C ABI
(``include/spattn.h``, ``libspattn.so``)."""
from .seqpar import *  # noqa: F401,F403
from . import losses  # noqa: F401
from .losses import *  # noqa: F401,F403
from .seqpar import (ConfigError, Fabric, RankContext, SequenceParallelAttention,  # noqa: F401
                     ShapeError, StateError, __version__, engine_attention, oracle_attention)
