"""Host twin of the device counter RNG (Philox4x32-10, A-15) for build-time draws
(camera randomisation).  Per-step draws (resets, benchmark actions) happen on the device
(csrc/sim_common.cuh); both use key = master seed, counter = (block, aux, global env, tag)."""

from __future__ import annotations

import numpy as np

_M0, _M1 = np.uint64(0xD2511F53), np.uint64(0xCD9E8D57)
_W0, _W1 = np.uint64(0x9E3779B9), np.uint64(0xBB67AE85)
_MASK = np.uint64(0xFFFFFFFF)

TAG_RESET = 0x52455354   # 'REST'
TAG_ACTION = 0x41435421  # 'ACT!'
TAG_CAMERA = 0x43414D52  # 'CAMR'


def philox4x32(c0, c1, c2, c3, seed: int):
    seed = int(seed) & 0xFFFFFFFFFFFFFFFF
    k0, k1 = np.uint64(seed & 0xFFFFFFFF), np.uint64(seed >> 32)
    c = [np.asarray(x, np.uint64) & _MASK for x in np.broadcast_arrays(c0, c1, c2, c3)]
    k0 = np.broadcast_to(k0, c[0].shape).copy()
    k1 = np.broadcast_to(k1, c[0].shape).copy()
    for r in range(10):
        if r:
            k0 = (k0 + _W0) & _MASK
            k1 = (k1 + _W1) & _MASK
        p0, p1 = _M0 * c[0], _M1 * c[2]
        c = [(p1 >> np.uint64(32)) ^ c[1] ^ k0, p1 & _MASK, (p0 >> np.uint64(32)) ^ c[3] ^ k1, p0 & _MASK]
    return c


def uniforms(seed: int, env_ids, aux: int, tag: int, n: int) -> np.ndarray:
    """(len(env_ids), n) float64 uniforms in [0, 1): block k -> draws 2k, 2k+1 with the 53-bit
    conversion ((a >> 5) * 2^26 + (b >> 6)) * 2^-53."""
    env_ids = np.asarray(env_ids, np.uint64)
    out = np.empty(env_ids.shape + (n,))
    for blk in range((n + 1) // 2):
        r = philox4x32(blk, aux, env_ids, tag, seed)
        for j in range(2):
            if 2 * blk + j < n:
                a, b = r[2 * j] >> np.uint64(5), r[2 * j + 1] >> np.uint64(6)
                out[..., 2 * blk + j] = (a * np.uint64(67108864) + b).astype(np.float64) * (1.0 / 9007199254740992.0)
    return out
