"""feinsum-B200: a B200-native evaluator for batched Einstein summations.

Host C++ (canonicalizer, planner, tuning facts) and sm_100a CUDA kernels live
in ``lib/libfeinsum_b200.so`` behind the C-ABI ``include/feinsum_b200.h``;
``feinsum`` is the Python mirror of the reference API over that ABI.
"""
from . import feinsum  # noqa: F401
from .feinsum import (FeinsumError, Plan, canonical_key, canonicalize, evaluate, evaluate_kernel,  # noqa: F401
                      is_isomorphic, parse_classic, print_classic, raise_kernel, identify_as_einsum, retrieve,
                      record_facts, validate)
