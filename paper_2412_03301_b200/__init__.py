"""B200-native hot path of BioVSS (arXiv 2412.03301): FlyHash + Bloom-sketch
filtered top-k vector-set search under the Hausdorff distance.

The compute lives in ``libbvss.so`` (hand-written sm_100a kernels behind the C
ABI in ``include/bvss.h``); ``bvss`` is its thin ctypes binding and ``dist``
the multi-GPU (one process per GPU) orchestration over torch.distributed.
"""
__all__ = ["bvss"]
