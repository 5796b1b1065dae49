"""Seeded synthetic workloads shared by the oracle tests, the GPU tests and
bench.py: info bits -> convolutional encoder -> puncturing -> BPSK/AWGN ->
int8 quantiser.  This module holds none of the decoder's arithmetic (no
branch metrics, no ACS, no traceback); it only produces inputs."""
from .channel import (CODES, PUNCT, CONFIGS, code_rate, sigma_for, info_bits, encode,
                      make_stream, make_window, llr_count, n_stages_of)

__all__ = ["CODES", "PUNCT", "CONFIGS", "code_rate", "sigma_for", "info_bits", "encode",
           "make_stream", "make_window", "llr_count", "n_stages_of"]
