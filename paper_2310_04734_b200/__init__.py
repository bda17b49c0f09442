"""paper_2310_04734_b200 — B200-native MOR frequency sweep (rational-Arnoldi ROM →
batched reduced sweep → cabin SPL) behind the reference `vibrofem` API.

Compute runs in libvibro_b200.so (hand-written sm_100a CUDA, C ABI in
include/vibro_b200.h).  There is no CPU fallback.
"""

__version__ = "0.1.0"
