"""B200-native out-of-core compressed stencil stepping (arXiv 2109.05410).

The compute path lives in the C-ABI library ``liboocz.so`` (CUDA, sm_100a);
``paper_2109_05410_b200.oocz`` is its thin ctypes binding.  ``synth`` holds the
seeded input generators shared with the tests.
"""
__all__ = ["oocz", "synth"]
