"""B200-native DASH optimizer step (arXiv 2602.02016): batched block-preconditioned Shampoo.

Drop-in for the reference ``blockshampoo`` package's optimizer and solver-selection API; every product,
solver iteration and update runs in hand-written sm_100a kernels behind the C ABI in
``include/dash_b200.h`` (``libdash_b200.so``).
"""
__version__ = "0.1.0"
