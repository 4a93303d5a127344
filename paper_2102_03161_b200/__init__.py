"""B200-native PipeTransformer hot path (arXiv 2102.03161).

The package holds the C-ABI library (libeps_b200.so: eps:: control plane +
sm_100a kernels), its ctypes binding and the host-side training loop.
"""
import os

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
# EPS_LIB_PATH points the binding at another build (A/B kernel comparisons in tools/)
LIB_PATH = os.environ.get("EPS_LIB_PATH") or os.path.join(PKG_DIR, "libeps_b200.so")
