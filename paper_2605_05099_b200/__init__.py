"""B200-native bulk stream fills with the reference `randstream` API.

    from paper_2605_05099_b200 import state_io
    r = state_io.create("x256**", seed=[2024])
    z = r.fill("norm", {}, 1 << 28)      # float64 CUDA tensor, bit-identical to the reference

Fills run as hand-written sm_100a CUDA kernels behind the C ABI in
include/randstream_b200.h (librandstream_b200.so); there is no CPU fallback.
"""

from . import _lib, engines, seeding, serialize, state_io  # noqa: F401
from .rng import Rng, fill_streams, semidefinite_factor  # noqa: F401
from .state_io import catalogue, create, duplicate, free, from_blob, last_error, to_blob  # noqa: F401

__version__ = "0.1.0"
