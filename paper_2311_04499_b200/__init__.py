"""B200-native COVAP gradient-synchronisation path (arXiv 2311.04499).

The product is ``libcovap_b200.so`` (sm_100a kernels + NCCL + host planner,
C-ABI in ``include/covap_c.h``); this package is its Python host mirror of
the reference API (``covap.py``; the baseline compressors under error
feedback in ``feedback.py``).  Importing it loads the shared library and
fails loudly when it is missing: there is no CPU fallback.
"""
from .errors import (ConfigError, CudaError, Error, IncompleteProfile, InvalidInput,  # noqa: F401
                     InvalidState, NcclError, NoDeviceError, UndefinedRatio)
from . import _lib  # noqa: F401
from .covap import *  # noqa: F401,F403
from .covap import (BucketPlan, CompressedUpdate, CompressorState, Communicator,  # noqa: F401
                    CovapConfig, CovapSync, EfSchedule, LayerSpec, ModelSpec, ProfileResult,
                    SelectionRule, allocate_buckets, allreduce_mean, ccr, choose_interval,
                    covap_compress, covap_decompress, ef_coefficient, effective_numels,
                    effective_tensors, generate, load_layout, median_numel, plan_for,
                    profile_ccr, select_tensors, shard_plan, spin, stream_key)
from . import feedback  # noqa: F401
from .feedback import (CovapFilter, ErrorFeedback, Fp16Filter, IdentityFilter,  # noqa: F401
                       RandomkFilter, TopkFilter, fp16_roundtrip, randomk_compress, sparsifier_k,
                       topk_compress)

_lib.lib()  # load now: a missing extension is an import error, not a silent fallback
