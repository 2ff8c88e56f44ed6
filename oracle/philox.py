"""Philox4x32-10 counter RNG in numpy (oracle twin of the device RNG) -- test infrastructure.

SPEC.md:221 requires per-env counter-based streams derived from (master_seed, env_index) so
partial resets are reproducible independent of other envs; A-15 fixes the
generator (Philox4x32-10, Salmon et al. SC'11) and the float conversions below.
"""

from __future__ import annotations

import numpy as np

M0, M1 = np.uint64(0xD2511F53), np.uint64(0xCD9E8D57)
W0, W1 = np.uint32(0x9E3779B9), np.uint32(0xBB67AE85)
MASK = np.uint64(0xFFFFFFFF)


def philox4x32(c0, c1, c2, c3, k0, k1, rounds: int = 10):
    """Vectorised Philox4x32-R; every argument is broadcast to a uint32 array."""
    c0, c1, c2, c3, k0, k1 = np.broadcast_arrays(*(np.asarray(x, dtype=np.uint64) & MASK
                                                   for x in (c0, c1, c2, c3, k0, k1)))
    c0, c1, c2, c3 = c0.copy(), c1.copy(), c2.copy(), c3.copy()
    k0, k1 = k0.copy(), k1.copy()
    for r in range(rounds):
        if r:
            k0 = (k0 + np.uint64(W0)) & MASK
            k1 = (k1 + np.uint64(W1)) & MASK
        p0 = M0 * c0
        p1 = M1 * c2
        hi0, lo0 = p0 >> np.uint64(32), p0 & MASK
        hi1, lo1 = p1 >> np.uint64(32), p1 & MASK
        c0, c1, c2, c3 = hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0
    return tuple(x.astype(np.uint32) for x in (c0, c1, c2, c3))


def u01_f64(a, b):
    """53-bit uniform in [0,1): ((a>>5)*2^26 + (b>>6)) * 2^-53 (exact in float64)."""
    a = np.asarray(a, np.uint64) >> np.uint64(5)
    b = np.asarray(b, np.uint64) >> np.uint64(6)
    return (a * np.uint64(67108864) + b).astype(np.float64) * (1.0 / 9007199254740992.0)


def u01_f32(a):
    """24-bit uniform in [0,1) as float32: (a>>8) * 2^-24."""
    return (np.asarray(a, np.uint32) >> np.uint32(8)).astype(np.float32) * np.float32(1.0 / 16777216.0)


def key_of(seed: int):
    seed = int(seed) & 0xFFFFFFFFFFFFFFFF
    return seed & 0xFFFFFFFF, seed >> 32


# Stream tags (counter word 3): keep the purposes of draws disjoint.
TAG_RESET = 0x52455354   # 'REST'
TAG_ACTION = 0x41435421  # 'ACT!'
TAG_CAMERA = 0x43414D52  # 'CAMR'


def reset_uniforms(seed: int, env_ids, reset_count, n: int):
    """n float64 uniforms per env for a reset: block k -> draws 2k, 2k+1.
    counter = (k, reset_count, global_env, TAG_RESET), key = seed."""
    env_ids = np.asarray(env_ids, dtype=np.uint64)
    rc = np.broadcast_to(np.asarray(reset_count, dtype=np.uint64), env_ids.shape)
    k0, k1 = key_of(seed)
    out = np.empty(env_ids.shape + (n,), dtype=np.float64)
    for blk in range((n + 1) // 2):
        r = philox4x32(blk, rc, env_ids, TAG_RESET, k0, k1)
        out[..., 2 * blk] = u01_f64(r[0], r[1])
        if 2 * blk + 1 < n:
            out[..., 2 * blk + 1] = u01_f64(r[2], r[3])
    return out


def uniform(lo, hi, u):
    """lo + (hi - lo) * u with separately rounded operations (no FMA)."""
    return lo + (hi - lo) * u


def action_uniforms(seed: int, step: int, env_ids, dim: int):
    """Random actions in [-1, 1) float32 for (step, env): counter = (blk, step, env, TAG_ACTION)."""
    env_ids = np.asarray(env_ids, dtype=np.uint64)
    k0, k1 = key_of(seed)
    out = np.empty(env_ids.shape + (dim,), dtype=np.float32)
    for blk in range((dim + 3) // 4):
        r = philox4x32(blk, step, env_ids, TAG_ACTION, k0, k1)
        for j in range(4):
            d = 4 * blk + j
            if d < dim:
                out[..., d] = u01_f32(r[j]) * np.float32(2.0) - np.float32(1.0)
    return out
