"""B200-native local-energy hot path of NNQS-Transformer (arXiv 2306.16705).

libnnqs.so (C-ABI, include/nnqs.h) holds every step of the path: host C++
Hamiltonian compression and sm_100a kernels for the lookup table, the
local energy and the energy reduction.  ``nnqs`` is the ctypes binding;
``distributed`` shards rows over GPUs with torch.distributed (NCCL).
"""
from .nnqs import *  # noqa: F401,F403
from .nnqs import EXPORTED, Hamiltonian, NNQSError, Table  # noqa: F401
