"""B200-native BitStack (arXiv 2410.23918) hot path: y = W_hat_n x from n stacked
~1-bit residual blocks, as hand-written sm_100a CUDA behind a C ABI
(include/bitstack.h).  Python here is argument marshalling only."""
from .bitstack import (  # noqa: F401
    BF16, F16, F32, BitStackError, Group, Layer, block_size_bits, compress, launch_count, load_library, matmul_grouped,
    profile_begin, profile_end, Store,
)
from . import budget  # noqa: F401,E402  (memory-budget level selection, host logic)
