"""B200-native LRQMM hot path (arXiv 2409.18772): liblrqmm.so + ctypes binding."""
from .lrqmm import (SIDE_A, SIDE_B, Lrqmm, LrqmmError, get_unique_id, load_library,  # noqa: F401
                    lrqmm_matmul)
