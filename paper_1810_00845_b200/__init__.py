"""B200-native hot path of CHET's encrypted tensor programs (arXiv 1810.00845).

``hisa``    -- binding of the C-ABI library libhisa.so (include/hisa.h): RNS-CKKS HISA
               instructions as sm_100a CUDA kernels (NTT/INTT, elementwise, key switching,
               rotation, relinearisation, rescale, samplers).
``driver``  -- HW-tiled CipherTensor metadata and the paper's tensor kernels (Alg. 1 conv,
               polynomial activation, average pooling, FC) issued through ``hisa``.
"""
__all__ = ["hisa"]
