"""paper_2502_06798_b200 -- B200-native (sm_100a) prompt-routing hot path of
"Prompt-Aware Scheduling for Efficient Text-to-Image Inferencing System" (arxiv 2502.06798).

The product is ``lib/libpas.so`` (C-ABI in ``include/pas.h``, CUDA sources in ``csrc/``);
``pas`` is its thin ctypes binding.  Import ``paper_2502_06798_b200.pas`` to use it -- it raises if
the library is not built (no CPU fallback).
"""
__all__ = ["pas", "build"]
