"""Seeded, counter-based value generator shared by the oracle and the bench/tests.

This module is INPUT GENERATION ONLY: it holds none of the method's arithmetic
(no attention, no tree, no density, no sharding).  Both sides of the parity
check draw their inputs from here (the CUDA filler in libblend implements the
same counter-based generator independently; tests compare the two bit-exactly).

Generator spec:

  mix(x)   = splitmix64(x)  (mod 2^64)
  H_j      = XOR_{i<=j} mix((tok_i << 32) ^ i ^ seed)          prefix hash of a token path
  KV[j,kvh,e] = grid(mix(H_j ^ mix(seed_kv + ((kind*2^8 + kvh)*2^12 + e))))   kind 0 = K, 1 = V
  Q[r,t,h,e]  = scale_q * grid(mix(seed_q ^ mix(((r*2^20 + t)*2^8 + h)*2^12 + e)))
  grid(z)  = ((z >> 56) - 128) / 128      256 levels in [-1, 1): exact in bf16 and fp32

K/V therefore depend only on the token prefix, so a shared prefix node has the
same K/V for every request through it by construction; the oracle never needs
the tree.  `r` is the GLOBAL request index, so sharded runs see identical Q.
"""
from __future__ import annotations

import numpy as np

M64 = np.uint64(0xFFFFFFFFFFFFFFFF)
_C0 = np.uint64(0x9E3779B97F4A7C15)
_C1 = np.uint64(0xBF58476D1CE4E5B9)
_C2 = np.uint64(0x94D049BB133111EB)

# derived seeds: seed_kv = seed ^ KV_SALT, seed_q = seed ^ Q_SALT
KV_SALT = 0x5BD1E9955BD1E995
Q_SALT = 0xC2B2AE3D27D4EB4F


def mix(x) -> np.ndarray:
    """splitmix64 finaliser on a uint64 array (wrapping arithmetic)."""
    z = np.asarray(x, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = z + _C0
        z = (z ^ (z >> np.uint64(30))) * _C1
        z = (z ^ (z >> np.uint64(27))) * _C2
        z = z ^ (z >> np.uint64(31))
    return z


def grid(z: np.ndarray) -> np.ndarray:
    """Top byte of z mapped to k/128 - 1, k in 0..255 (exact in bf16/fp32)."""
    return ((z >> np.uint64(56)).astype(np.int64) - 128).astype(np.float64) / 128.0


def prefix_hash(tokens: np.ndarray, seed: int) -> np.ndarray:
    """H_j for j = 0..n-1 of one token path (uint64[n])."""
    tok = np.asarray(tokens, dtype=np.int64).astype(np.uint64)
    pos = np.arange(tok.shape[0], dtype=np.uint64)
    leaf = mix((tok << np.uint64(32)) ^ pos ^ np.uint64(seed & 0xFFFFFFFFFFFFFFFF))
    return np.bitwise_xor.accumulate(leaf) if leaf.size else leaf


def kv_salt_table(seed: int, kind: int, num_kv_heads: int, head_dim: int, kv_head0: int = 0) -> np.ndarray:
    """mix(seed_kv + ((kind*2^8 + kvh)*2^12 + e)) as uint64[Hkv, D], kvh = kv_head0 .. +Hkv-1
    (global kv head indices: a head-parallel slice keeps the full problem's values)."""
    seed_kv = np.uint64((seed ^ KV_SALT) & 0xFFFFFFFFFFFFFFFF)
    kvh = np.arange(kv_head0, kv_head0 + num_kv_heads, dtype=np.uint64)[:, None]
    e = np.arange(head_dim, dtype=np.uint64)[None, :]
    ctr = ((np.uint64(kind) << np.uint64(8)) + kvh) * np.uint64(1 << 12) + e
    with np.errstate(over="ignore"):
        return mix(seed_kv + ctr)


def kv_values(h: np.ndarray, seed: int, kind: int, num_kv_heads: int, head_dim: int,
              kv_head0: int = 0) -> np.ndarray:
    """K (kind=0) or V (kind=1) values float64[n, Hkv, D] for prefix hashes h[n]."""
    salt = kv_salt_table(seed, kind, num_kv_heads, head_dim, kv_head0)
    z = mix(np.asarray(h, dtype=np.uint64)[:, None, None] ^ salt[None, :, :])
    return grid(z)


def path_kv(tokens: np.ndarray, seed: int, num_kv_heads: int, head_dim: int, kv_head0: int = 0):
    """(K, V) float64[n, Hkv, D] of a full token path."""
    h = prefix_hash(tokens, seed)
    return (kv_values(h, seed, 0, num_kv_heads, head_dim, kv_head0),
            kv_values(h, seed, 1, num_kv_heads, head_dim, kv_head0))


def q_values(global_req: int, t: np.ndarray, seed: int, num_q_heads: int, head_dim: int,
             scale_q: float = 1.0, head0: int = 0) -> np.ndarray:
    """Q float64[len(t), Hq, D] for query indices t of request `global_req`, q heads
    head0 .. head0+Hq-1 (global head indices)."""
    seed_q = np.uint64((seed ^ Q_SALT) & 0xFFFFFFFFFFFFFFFF)
    t = np.asarray(t, dtype=np.uint64)[:, None, None]
    h = np.arange(head0, head0 + num_q_heads, dtype=np.uint64)[None, :, None]
    e = np.arange(head_dim, dtype=np.uint64)[None, None, :]
    with np.errstate(over="ignore"):
        ctr = ((np.uint64(global_req) * np.uint64(1 << 20) + t) * np.uint64(1 << 8) + h) \
            * np.uint64(1 << 12) + e
        z = mix(seed_q ^ mix(ctr))
    return scale_q * grid(z)


def segment_hash(tokens: np.ndarray, start: int, h_prev: int, seed: int) -> np.ndarray:
    """H_j for j = start .. start+len(tokens)-1 of a path whose prefix hash at
    position start-1 is h_prev (0 for start = 0): the per-node form of prefix_hash."""
    tok = np.asarray(tokens, dtype=np.int64).astype(np.uint64)
    pos = np.arange(start, start + tok.shape[0], dtype=np.uint64)
    leaf = mix((tok << np.uint64(32)) ^ pos ^ np.uint64(seed & 0xFFFFFFFFFFFFFFFF))
    if leaf.size == 0:
        return leaf
    return np.bitwise_xor.accumulate(leaf) ^ np.uint64(h_prev)
