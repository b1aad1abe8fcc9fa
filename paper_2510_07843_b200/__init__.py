"""B200-native per-RE MMSE MIMO detector + max-log soft demapper (arxiv 2510.07843 hot path).

Product path: hand-written sm_100a CUDA kernels behind the C ABI in include/mimo.h
(libmimo.so, built in-tree by `python -m paper_2510_07843_b200.build`), with a thin
ctypes binding in `paper_2510_07843_b200.mimo`. There is no CPU fallback: if
libmimo.so is missing or no CUDA device is present, the binding raises.
"""
__all__ = ["mimo", "synth"]
