"""Oracle EpisodeMetrics -- test infrastructure (oracle/__init__.py).

Per env: return = sum of the step rewards (float64 accumulation of the float32 rewards, in
step order), length = steps in the episode, success_once / fail_once latch on the first
success / fail, success_at_end / fail_at_end are the flags of the final step.  A record is
emitted when the episode ends (terminated or truncated) and the accumulators restart.
"""

from __future__ import annotations

import numpy as np


def reference_metrics(success, fail, rewards):
    """Definition for one finished episode given its per-step flag/reward sequences."""
    success, fail = np.asarray(success, bool), np.asarray(fail, bool)
    ret = 0.0
    for r in rewards:
        ret = ret + float(np.float32(r))
    return {"return": ret, "length": len(success), "success_once": bool(success.any()),
            "success_at_end": bool(success[-1]), "fail_once": bool(fail.any()), "fail_at_end": bool(fail[-1])}


class EpisodeAccumulator:
    def __init__(self, B):
        self.ret = np.zeros(B)
        self.so = np.zeros(B, bool)
        self.fo = np.zeros(B, bool)

    def reset(self, mask=None):
        m = slice(None) if mask is None else mask
        self.ret[m] = 0.0
        self.so[m] = False
        self.fo[m] = False

    def update(self, reward, success, fail, terminated, truncated, length):
        """Returns (done mask, return, length, flags u8) like the device outputs."""
        ret = self.ret + np.asarray(reward, np.float32).astype(np.float64)
        so = self.so | success
        fo = self.fo | fail
        done = terminated | truncated
        flags = (so.astype(np.uint8) | (success.astype(np.uint8) << 1) | (fo.astype(np.uint8) << 2)
                 | (fail.astype(np.uint8) << 3))
        out = (done.copy(), np.where(done, ret, 0.0), np.where(done, length, 0), np.where(done, flags, 0))
        self.ret = np.where(done, 0.0, ret)
        self.so = np.where(done, False, so)
        self.fo = np.where(done, False, fo)
        return out
