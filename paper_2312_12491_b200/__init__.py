"""B200-native streaming denoise loop (StreamDiffusion, arXiv 2312.12491).

The hot path is libstagger_b200.so (sm_100a kernels behind the C-ABI in
include/stagger_b200.h); this package holds its build recipe and the Python
mirror of the reference `stagger` operator API (stagger.py)."""
import os

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG_DIR, "libstagger_b200.so")


def load():
    """Import the ctypes binding (raises if the CUDA library is missing)."""
    from . import stagger  # noqa: F401

    return stagger
