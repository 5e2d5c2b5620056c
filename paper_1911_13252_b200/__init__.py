"""B200-native ELM training of recurrent networks (arXiv 1911.13252).

The product is the C-ABI library ``libelmrnn.so`` (include/elmrnn.h) built
from ``csrc/`` for sm_100a; ``elmrnn`` is its thin Python binding and
``parallel`` the row-sharded multi-GPU driver over torch.distributed.
"""
from .elmrnn import ARCHS, ELMRNN, ElmrnnError, SolveInfo, lib  # noqa: F401
