"""numpy Philox4x32-10 (Salmon, Moraes, Dror, Shaw, SC'11; Random123).

Test infrastructure. Restates paper_2512_09664_b200/csrc/common.cuh
philox4x32_10/draw so generated particle arrays can be checked bit-exactly.
The reference's own RNG (rng.py:33-106, splitmix64) is NOT reproduced by the
B200 generator; oracle mode injects reference particles instead.

Pinned by tests/test_oracle_philox.py against Random123's published
known-answer vectors and NVIDIA's curand_Philox4x32_10 (host build).
"""

from __future__ import annotations

import numpy as np

M0 = np.uint64(0xD2511F53)
M1 = np.uint64(0xCD9E8D57)
W0 = 0x9E3779B9
W1 = 0xBB67AE85
MASK32 = np.uint64(0xFFFFFFFF)

TAG_PARTICLE_A = 0x01
TAG_PARTICLE_B = 0x02
TAG_PERTURB = 0x03
TAG_PAIR = 0x04
TAG_NOISE = 0x10
TAG_CELL = 0x20

# Random123 kat_vectors, philox4x32 R=10: (counter[4], key[2]) -> out[4]
KAT = [
    ((0x00000000, 0x00000000, 0x00000000, 0x00000000), (0x00000000, 0x00000000),
     (0x6627e8d5, 0xe169c58d, 0xbc57ac4c, 0x9b00dbd8)),
    ((0xffffffff, 0xffffffff, 0xffffffff, 0xffffffff), (0xffffffff, 0xffffffff),
     (0x408f276d, 0x41c83b0e, 0xa20bc7c6, 0x6d5451fd)),
    ((0x243f6a88, 0x85a308d3, 0x13198a2e, 0x03707344), (0xa4093822, 0x299f31d0),
     (0xd16cfe09, 0x94fdcceb, 0x5001e420, 0x24126ea1)),
]


def philox4x32_10(c0, c1, c2, c3, k0: int, k1: int):
    """Vectorised Philox4x32-10. Counters: uint32-valued arrays (broadcast)."""
    c0 = np.asarray(c0, dtype=np.uint64) & MASK32
    c1 = np.asarray(c1, dtype=np.uint64) & MASK32
    c2 = np.asarray(c2, dtype=np.uint64) & MASK32
    c3 = np.asarray(c3, dtype=np.uint64) & MASK32
    c0, c1, c2, c3 = np.broadcast_arrays(c0, c1, c2, c3)
    k0 = int(k0) & 0xFFFFFFFF
    k1 = int(k1) & 0xFFFFFFFF
    for _ in range(10):
        p0 = M0 * c0
        p1 = M1 * c2
        hi0, lo0 = p0 >> np.uint64(32), p0 & MASK32
        hi1, lo1 = p1 >> np.uint64(32), p1 & MASK32
        c0, c1, c2, c3 = (hi1 ^ c1 ^ np.uint64(k0), lo1, hi0 ^ c3 ^ np.uint64(k1), lo0)
        k0 = (k0 + W0) & 0xFFFFFFFF
        k1 = (k1 + W1) & 0xFFFFFFFF
    return c0.astype(np.uint32), c1.astype(np.uint32), c2.astype(np.uint32), c3.astype(np.uint32)


def draw(seed: int, gpair: int, batch: int, index, tag: int):
    """Four words of stream `tag` at counter (index, pair, batch, tag)."""
    seed = int(seed) & 0xFFFFFFFFFFFFFFFF
    return philox4x32_10(index, gpair, batch & 0xFFFFFFFF, tag, seed & 0xFFFFFFFF, seed >> 32)


def u32_to_unit(w) -> np.ndarray:
    """(w + 0.5) * 2^-32, exact in float64 (common.cuh u32_to_unit)."""
    return (np.asarray(w, dtype=np.float64) + 0.5) * 2.0 ** -32


def u53_to_unit(lo, hi) -> np.ndarray:
    bits = ((np.asarray(hi, dtype=np.uint64) << np.uint64(32)) | np.asarray(lo, dtype=np.uint64)) >> np.uint64(11)
    return (bits.astype(np.float64) + 0.5) * 2.0 ** -53


def u32_to_unitf(w) -> np.ndarray:
    """23-bit float32 uniform ((w >> 9) + 0.5) * 2^-23, exact and open in float32."""
    w = np.asarray(w, dtype=np.uint32)
    return ((w >> np.uint32(9)).astype(np.float32) + np.float32(0.5)) * np.float32(2.0 ** -23)


def u32_to_radius_unitf(w) -> np.ndarray:
    """Box-Muller radius uniform of the GPU (common.cuh box_muller):
    f32(f32(w) * 2^-32 + 2^-33), one rounding (exact in float64 before it), in (0, 1]."""
    w = np.asarray(w, dtype=np.uint32)
    return (w.astype(np.float32).astype(np.float64) * 2.0 ** -32 + 2.0 ** -33).astype(np.float32)


def box_muller64(wa, wb):
    """Float64 Box-Muller on the same uniforms as the GPU (32-bit radius
    uniform, 23-bit angle uniform; the GPU uses MUFU approximations, so
    agreement is to ~1e-6, not bit-exact)."""
    u1 = u32_to_radius_unitf(wa).astype(np.float64)
    u2 = u32_to_unitf(wb).astype(np.float64)
    r = np.sqrt(-2.0 * np.log(u1))
    t = 2.0 * np.pi * u2
    return r * np.cos(t), r * np.sin(t)
