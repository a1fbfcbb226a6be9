"""B200-native vertex-star Schwarz smoother / V-cycle of arXiv 2104.14855.

The product is libmhdp.so (CUDA kernels for sm_100a + C-ABI, include/mhdp.h);
`mhdp` is its thin ctypes binding, `workloads` names the BASELINE.json configurations
and draws their seeded synthetic inputs.
"""
