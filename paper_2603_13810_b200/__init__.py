"""B200-native Conv-LIF hot path of arXiv 2603.13810 (TAC / TAC-TP / dense).

The compute lives in libtacsnn.so (hand-written sm_100a kernels behind the C ABI
of include/tacsnn.h); ``tacsnn`` is its ctypes binding, ``network`` stacks layers,
``synth`` generates seeded synthetic inputs, ``configs`` names the BASELINE
workloads.  Modules are imported lazily so that the input generators can be used
without loading the CUDA library.
"""
__all__ = ["tacsnn", "network", "synth", "configs", "build"]
