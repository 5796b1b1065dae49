"""B200-native parallel block-based Viterbi decoder (PBVD) after Peng et al.,
arXiv 1608.00066.  The hot path lives in libpbvd.so (sm_100a CUDA kernels
behind the C ABI of include/pbvd.h); this package is its thin Python binding
plus the multi-GPU sharding driver."""
from .decoder import (Decoder, PbvdError, StreamDecoder, jit_prebuild, probe_acs_balanced,
                      probe_acs_peak, supported)

__all__ = ["Decoder", "PbvdError", "StreamDecoder", "jit_prebuild", "probe_acs_balanced",
           "probe_acs_peak", "supported"]
