"""Minimal PPO over the device env protocol (the ``learn`` module; PAPER.md 4.3).

This is the consumer downstream of the hot path: rollouts read the fused step kernel's device
observations, rewards and flags directly, with no host round trip.  Everything stays on the
GPU: the policy forward pass, Gaussian sampling, GAE, the hand-derived backward pass and Adam.

* ``PolicyNet``: a two-hidden-layer (width 64, tanh) MLP with a Gaussian head and a
  state-independent log-std.  The value head is either a separate MLP of the same shape or a
  linear head on the shared trunk (``shared_trunk``).  Gradients come from hand-derived
  layer backward rules (``PolicyNet.backward``), with no autodiff.  They are checked against
  central finite differences at fp64 (tests/test_learn.py).
* ``compute_gae``: the standard GAE recursion, time-major; a done at t cuts bootstrapping.
  ``normalize_advantages`` gives mean 0 and std 1 per update.
* ``ppo_loss``: the clipped surrogate, the clipped value loss and the entropy bonus, with
  gradients with respect to (mu, log_std, v).
* ``ppo_train(env, cfg, seed)``: rollout -> GAE -> epochs x minibatches of Adam steps with a
  global grad-norm clip.  Observation normalisation uses running mean/var (Welford / Chan),
  frozen at eval.  Eval runs through ``metrics.eval_wrapper`` at intervals.  The log records
  wall-clock per phase (rollout vs update) and env-step accounting (num_envs x rollout_len x
  iterations exactly).  A NaN loss aborts with a diagnostic dump.
"""

from __future__ import annotations

import math
import time
from dataclasses import dataclass, field
from typing import Dict, List, Optional

import torch

LOG_2PI = math.log(2.0 * math.pi)


@dataclass
class PPOConfig:
    num_envs: int = 1024
    rollout_len: int = 32
    epochs: int = 4
    minibatches: int = 4
    clip_eps: float = 0.2
    gamma: float = 0.99
    gae_lambda: float = 0.95
    lr: float = 1e-3
    vf_coef: float = 0.5
    ent_coef: float = 0.0
    max_grad_norm: float = 0.5
    total_steps: int = 2_000_000
    eval_interval: int = 10        # iterations between evaluations (0 = only at the end)
    eval_envs: int = 256
    hidden: int = 64
    shared_trunk: bool = False
    init_log_std: float = -0.5
    obs_clip: float = 10.0

    def __post_init__(self):
        for k in ("num_envs", "rollout_len", "epochs", "minibatches", "lr", "total_steps", "hidden", "eval_envs"):
            if not getattr(self, k) > 0:
                raise ValueError(f"PPOConfig.{k} must be positive")
        if not 0.0 < self.clip_eps < 1.0:
            raise ValueError("PPOConfig.clip_eps must lie in (0, 1)")
        for k in ("gamma", "gae_lambda"):
            if not 0.0 <= getattr(self, k) <= 1.0:
                raise ValueError(f"PPOConfig.{k} must lie in [0, 1]")


# ----------------------------------------------------------------------------- the network
class PolicyNet:
    """Two tanh hidden layers of width `hidden`; Gaussian mean head; state-independent log-std;
    value head separate (default) or on the shared trunk.  Parameters live in `self.p`."""

    def __init__(self, obs_dim: int, act_dim: int, hidden: int = 64, shared_trunk: bool = False,
                 seed: int = 0, device=None, dtype=torch.float32, init_log_std: float = -0.5):
        self.obs_dim, self.act_dim, self.hidden, self.shared = obs_dim, act_dim, hidden, shared_trunk
        g = torch.Generator(device="cpu").manual_seed(int(seed))

        def lin(fan_in, fan_out, gain):
            w = torch.randn((fan_in, fan_out), generator=g, dtype=torch.float64) * (gain / math.sqrt(fan_in))
            return w.to(device=device, dtype=dtype), torch.zeros(fan_out, device=device, dtype=dtype)

        p = {}
        p["W1"], p["b1"] = lin(obs_dim, hidden, math.sqrt(2.0))
        p["W2"], p["b2"] = lin(hidden, hidden, math.sqrt(2.0))
        p["W3"], p["b3"] = lin(hidden, act_dim, 0.01)
        p["log_std"] = torch.full((act_dim,), float(init_log_std), device=device, dtype=dtype)
        if shared_trunk:
            p["Vh"], p["ch"] = lin(hidden, 1, 1.0)
        else:
            p["V1"], p["c1"] = lin(obs_dim, hidden, math.sqrt(2.0))
            p["V2"], p["c2"] = lin(hidden, hidden, math.sqrt(2.0))
            p["V3"], p["c3"] = lin(hidden, 1, 1.0)
        self.p: Dict[str, torch.Tensor] = p

    def num_params(self) -> int:
        return sum(t.numel() for t in self.p.values())

    def forward(self, x: torch.Tensor):
        p = self.p
        h1 = torch.tanh(torch.addmm(p["b1"], x, p["W1"]))
        h2 = torch.tanh(torch.addmm(p["b2"], h1, p["W2"]))
        mu = torch.addmm(p["b3"], h2, p["W3"])
        if self.shared:
            v = torch.addmm(p["ch"], h2, p["Vh"]).squeeze(-1)
            cache = (x, h1, h2)
        else:
            g1 = torch.tanh(torch.addmm(p["c1"], x, p["V1"]))
            g2 = torch.tanh(torch.addmm(p["c2"], g1, p["V2"]))
            v = torch.addmm(p["c3"], g2, p["V3"]).squeeze(-1)
            cache = (x, h1, h2, g1, g2)
        return mu, p["log_std"], v, cache

    def backward(self, cache, d_mu: torch.Tensor, d_log_std: torch.Tensor, d_v: torch.Tensor) -> Dict[str, torch.Tensor]:
        """Hand-derived reverse pass: dL/dparams from dL/dmu (B, A), dL/dlog_std (A), dL/dv (B)."""
        p = self.p
        gr = {"log_std": d_log_std}
        x, h1, h2 = cache[0], cache[1], cache[2]
        dv = d_v.unsqueeze(-1)
        gr["W3"] = h2.t() @ d_mu
        gr["b3"] = d_mu.sum(0)
        d_h2 = d_mu @ p["W3"].t()
        if self.shared:
            gr["Vh"] = h2.t() @ dv
            gr["ch"] = dv.sum(0)
            d_h2 = d_h2 + dv @ p["Vh"].t()
        else:
            g1, g2 = cache[3], cache[4]
            gr["V3"] = g2.t() @ dv
            gr["c3"] = dv.sum(0)
            d_a2 = (dv @ p["V3"].t()) * (1.0 - g2 * g2)
            gr["V2"] = g1.t() @ d_a2
            gr["c2"] = d_a2.sum(0)
            d_a1 = (d_a2 @ p["V2"].t()) * (1.0 - g1 * g1)
            gr["V1"] = x.t() @ d_a1
            gr["c1"] = d_a1.sum(0)
        d_a2 = d_h2 * (1.0 - h2 * h2)
        gr["W2"] = h1.t() @ d_a2
        gr["b2"] = d_a2.sum(0)
        d_a1 = (d_a2 @ p["W2"].t()) * (1.0 - h1 * h1)
        gr["W1"] = x.t() @ d_a1
        gr["b1"] = d_a1.sum(0)
        return gr


def gaussian_logp(a: torch.Tensor, mu: torch.Tensor, log_std: torch.Tensor) -> torch.Tensor:
    z = (a - mu) * torch.exp(-log_std)
    return -0.5 * (z * z).sum(-1) - log_std.sum() - 0.5 * a.shape[-1] * LOG_2PI


def gaussian_entropy(log_std: torch.Tensor) -> torch.Tensor:
    return (log_std + 0.5 * (1.0 + LOG_2PI)).sum()


# ----------------------------------------------------------------------------- PPO pieces
def compute_gae(rewards, values, dones, last_value, gamma: float, lam: float):
    """Time-major (T, N) arrays.  dones[t] = the episode ended at step t, so V(s_{t+1}) is not
    bootstrapped.  Returns (advantages, returns) before normalisation."""
    rewards, values, dones = (torch.as_tensor(x) for x in (rewards, values, dones))
    if rewards.shape != values.shape or rewards.shape != dones.shape:
        raise ValueError(f"shape mismatch: rewards {tuple(rewards.shape)}, values {tuple(values.shape)}, "
                         f"dones {tuple(dones.shape)}")
    last_value = torch.as_tensor(last_value, dtype=values.dtype, device=values.device)
    if last_value.shape != rewards.shape[1:]:
        raise ValueError(f"last_value shape {tuple(last_value.shape)} != {tuple(rewards.shape[1:])}")
    T = rewards.shape[0]
    adv = torch.zeros_like(values)
    nxt_adv = torch.zeros_like(last_value)
    nxt_val = last_value
    for t in range(T - 1, -1, -1):
        live = 1.0 - dones[t].to(values.dtype)
        delta = rewards[t] + gamma * nxt_val * live - values[t]
        nxt_adv = delta + gamma * lam * live * nxt_adv
        adv[t] = nxt_adv
        nxt_val = values[t]
    return adv, adv + values


def normalize_advantages(adv: torch.Tensor) -> torch.Tensor:
    return (adv - adv.mean()) / (adv.std(unbiased=False) + 1e-12)


def ppo_loss(mu, log_std, v, batch: dict, clip_eps: float, vf_coef: float, ent_coef: float):
    """Clipped surrogate + clipped value loss - entropy bonus (means over the minibatch) and
    its gradients with respect to (mu, log_std, v)."""
    a, logp_old, adv, ret, v_old = batch["act"], batch["logp"], batch["adv"], batch["ret"], batch["val"]
    B = a.shape[0]
    inv_std = torch.exp(-log_std)
    z = (a - mu) * inv_std
    logp = -0.5 * (z * z).sum(-1) - log_std.sum() - 0.5 * a.shape[-1] * LOG_2PI
    ratio = torch.exp(logp - logp_old)
    clipped = ratio.clamp(1.0 - clip_eps, 1.0 + clip_eps)
    s1, s2 = ratio * adv, clipped * adv
    pg = -torch.minimum(s1, s2).mean()
    # d(-min(s1, s2))/dlogp: the unclipped branch when it is the min, else the clipped branch
    # (whose derivative is zero outside [1-eps, 1+eps])
    inside = (ratio >= 1.0 - clip_eps) & (ratio <= 1.0 + clip_eps)
    use1 = s1 <= s2
    d_logp = -(adv * ratio) * (use1 | inside).to(mu.dtype) / B
    vc = v_old + (v - v_old).clamp(-clip_eps, clip_eps)
    e1, e2 = (v - ret) ** 2, (vc - ret) ** 2
    vl = 0.5 * torch.maximum(e1, e2).mean()
    vin = ((v - v_old).abs() <= clip_eps).to(v.dtype)
    d_v = vf_coef * torch.where(e1 >= e2, v - ret, (vc - ret) * vin) / B
    ent = gaussian_entropy(log_std)
    loss = pg + vf_coef * vl - ent_coef * ent
    # logp = -0.5 |z|^2 - sum(log_std) - const:  dlogp/dmu = z / std,  dlogp/dlog_std = z^2 - 1
    d_mu = d_logp.unsqueeze(-1) * z * inv_std
    d_log_std = (d_logp.unsqueeze(-1) * (z * z - 1.0)).sum(0) - ent_coef * torch.ones_like(log_std)
    with torch.no_grad():
        approx_kl = ((ratio - 1.0) - (logp - logp_old)).mean()
        clip_frac = (~inside).to(torch.float32).mean()
    stats = {"loss": loss, "pg_loss": pg, "v_loss": vl, "entropy": ent, "approx_kl": approx_kl,
             "clip_frac": clip_frac}
    return stats, d_mu, d_log_std, d_v


class RunningMeanStd:
    """Running mean/var of observations (Chan et al. parallel update); frozen at eval."""

    def __init__(self, dim, device, dtype=torch.float64):
        self.mean = torch.zeros(dim, device=device, dtype=dtype)
        self.var = torch.ones(dim, device=device, dtype=dtype)
        self.count = torch.zeros((), device=device, dtype=dtype)
        self.frozen = False

    def update(self, x: torch.Tensor) -> None:
        if self.frozen:
            return
        x = x.to(self.mean.dtype)
        bm, bv, n = x.mean(0), x.var(0, unbiased=False), x.shape[0]
        tot = self.count + n
        d = bm - self.mean
        self.mean = self.mean + d * (n / tot)
        self.var = (self.var * self.count + bv * n + d * d * (self.count * n / tot)) / tot
        self.count = tot

    def normalize(self, x: torch.Tensor, clip: float = 10.0) -> torch.Tensor:
        y = (x - self.mean.to(x.dtype)) * torch.rsqrt(self.var.to(x.dtype) + 1e-8)
        return y.clamp(-clip, clip)


class Adam:
    def __init__(self, params: Dict[str, torch.Tensor], lr: float, betas=(0.9, 0.999), eps: float = 1e-8):
        self.p, self.lr, self.b1, self.b2, self.eps, self.t = params, lr, betas[0], betas[1], eps, 0
        self.m = {k: torch.zeros_like(v) for k, v in params.items()}
        self.v = {k: torch.zeros_like(v) for k, v in params.items()}

    def step(self, grads: Dict[str, torch.Tensor]) -> None:
        self.t += 1
        c1, c2 = 1.0 - self.b1 ** self.t, 1.0 - self.b2 ** self.t
        for k, g in grads.items():
            m, v = self.m[k], self.v[k]
            m.mul_(self.b1).add_(g, alpha=1.0 - self.b1)
            v.mul_(self.b2).addcmul_(g, g, value=1.0 - self.b2)
            self.p[k].addcdiv_(m, (v / c2).sqrt_().add_(self.eps), value=-self.lr / c1)


def clip_grad_norm(grads: Dict[str, torch.Tensor], max_norm: float) -> torch.Tensor:
    total = torch.sqrt(sum((g.double() * g.double()).sum() for g in grads.values()))
    scale = torch.clamp(max_norm / (total + 1e-6), max=1.0)
    for g in grads.values():
        g.mul_(scale.to(g.dtype))
    return total


# ----------------------------------------------------------------------------- train / eval
@dataclass
class TrainLog:
    iterations: List[dict] = field(default_factory=list)
    evals: List[dict] = field(default_factory=list)
    env_steps: int = 0
    rollout_seconds: float = 0.0
    update_seconds: float = 0.0


def evaluate(env, net: PolicyNet, rms: RunningMeanStd, seed: int = 12345) -> dict:
    """Deterministic (mean-action) episodes through metrics.eval_wrapper: every env runs to
    its time limit; returns mean return, success_at_end and success_once rates."""
    from .metrics import episode_records, eval_wrapper

    eval_wrapper(env)
    obs = env.reset(seed=seed)
    T = int(env.c_params.max_steps)
    rec = None
    for _ in range(T):
        mu, _, _, _ = net.forward(rms.normalize(obs.to(net.p["W1"].dtype)))
        r = env.step(mu.clamp(-1.0, 1.0).to(torch.float32).contiguous())
        obs = r.obs
        rec = episode_records(r.info)
    done = rec["done"]
    n = max(int(done.sum().item()), 1)
    return {"episodes": int(done.sum().item()),
            "return": float((rec["return"] * done).sum().item() / n),
            "success_at_end": float((rec["success_at_end"] & done).sum().item() / n),
            "success_once": float((rec["success_once"] & done).sum().item() / n)}


def ppo_train(env, cfg: PPOConfig, seed: int = 0, eval_env=None, time_limit: Optional[float] = None,
              log_fn=None, target_success: Optional[float] = None):
    """Train a PolicyNet on `env` (state obs, continuous actions).  Returns (net, rms, log)."""
    dev = env.device
    dtype = torch.float32
    if env.num_envs != cfg.num_envs:
        raise ValueError(f"env has {env.num_envs} envs, config says {cfg.num_envs}")
    net = PolicyNet(env.obs_dim, env.action_dim, cfg.hidden, cfg.shared_trunk, seed, dev, dtype, cfg.init_log_std)
    opt = Adam(net.p, cfg.lr)
    rms = RunningMeanStd(env.obs_dim, dev)
    gen = torch.Generator(device=dev).manual_seed(int(seed))
    N, T, A = env.num_envs, cfg.rollout_len, env.action_dim
    buf_obs = torch.zeros((T, N, env.obs_dim), device=dev, dtype=dtype)
    buf_act = torch.zeros((T, N, A), device=dev, dtype=dtype)
    buf_logp = torch.zeros((T, N), device=dev, dtype=dtype)
    buf_rew = torch.zeros((T, N), device=dev, dtype=dtype)
    buf_done = torch.zeros((T, N), device=dev, dtype=dtype)
    buf_val = torch.zeros((T, N), device=dev, dtype=dtype)
    iters = max(1, math.ceil(cfg.total_steps / (N * T)))
    log = TrainLog()
    obs = env.reset(seed=seed)
    t_start = time.perf_counter()
    for it in range(iters):
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        for t in range(T):
            rms.update(obs)
            o = rms.normalize(obs.to(dtype), cfg.obs_clip)
            mu, log_std, v, _ = net.forward(o)
            a = mu + torch.exp(log_std) * torch.randn(mu.shape, generator=gen, device=dev, dtype=dtype)
            buf_obs[t], buf_act[t], buf_logp[t], buf_val[t] = o, a, gaussian_logp(a, mu, log_std), v
            r = env.step(a.clamp(-1.0, 1.0).contiguous())
            buf_rew[t] = r.reward
            buf_done[t] = (r.terminated | r.truncated).to(dtype)
            # a time-limit truncation is not a terminal state: bootstrap gamma * V(s_T) from the
            # observation the episode ended in (the kernel exports it before the auto-reset)
            trunc = (r.truncated.bool() & ~r.terminated.bool()).to(dtype)
            _, _, v_fin, _ = net.forward(rms.normalize(r.info["final_obs"].to(dtype), cfg.obs_clip))
            buf_rew[t] += cfg.gamma * v_fin * trunc
            obs = r.obs
        _, _, last_v, _ = net.forward(rms.normalize(obs.to(dtype), cfg.obs_clip))
        adv, ret = compute_gae(buf_rew, buf_val, buf_done, last_v, cfg.gamma, cfg.gae_lambda)
        torch.cuda.synchronize(dev)
        t1 = time.perf_counter()
        flat = {"obs": buf_obs.reshape(T * N, -1), "act": buf_act.reshape(T * N, -1), "logp": buf_logp.reshape(-1),
                "adv": normalize_advantages(adv.reshape(-1)), "ret": ret.reshape(-1), "val": buf_val.reshape(-1)}
        mb = (T * N) // cfg.minibatches
        stats = None
        for _ in range(cfg.epochs):
            perm = torch.randperm(T * N, generator=gen, device=dev)
            for k in range(cfg.minibatches):
                idx = perm[k * mb:(k + 1) * mb]
                batch = {key: val.index_select(0, idx) for key, val in flat.items()}
                mu, log_std, v, cache = net.forward(batch["obs"])
                stats, d_mu, d_ls, d_v = ppo_loss(mu, log_std, v, batch, cfg.clip_eps, cfg.vf_coef, cfg.ent_coef)
                grads = net.backward(cache, d_mu, d_ls, d_v)
                gnorm = clip_grad_norm(grads, cfg.max_grad_norm)
                opt.step(grads)
        torch.cuda.synchronize(dev)
        t2 = time.perf_counter()
        rec = {k: float(v.item()) for k, v in stats.items()}
        if not all(math.isfinite(x) for x in rec.values()):
            raise FloatingPointError(f"PPO loss is not finite at iteration {it}: {rec}; grad norm "
                                     f"{float(gnorm)}; log_std {net.p['log_std'].tolist()}; obs mean "
                                     f"{rms.mean.tolist()}")
        log.env_steps += N * T
        log.rollout_seconds += t1 - t0
        log.update_seconds += t2 - t1
        rec.update(iteration=it, env_steps=log.env_steps, rollout_s=t1 - t0, update_s=t2 - t1,
                   mean_reward=float(buf_rew.mean().item()), grad_norm=float(gnorm))
        log.iterations.append(rec)
        last = it == iters - 1 or (time_limit is not None and time.perf_counter() - t_start > time_limit)
        if eval_env is not None and (last or (cfg.eval_interval and (it + 1) % cfg.eval_interval == 0)):
            rms.frozen = True
            ev = evaluate(eval_env, net, rms)
            rms.frozen = False
            ev.update(iteration=it, env_steps=log.env_steps, wall_s=time.perf_counter() - t_start)
            log.evals.append(ev)
            if log_fn:
                log_fn(ev)
            if target_success is not None and ev["success_at_end"] >= target_success:
                break
        if log_fn:
            log_fn(rec)
        if last:
            break
    return net, rms, log


def main(argv=None) -> int:
    """CLI: python -m paper_2410_00425_b200.learn --task CartpoleBalance --envs 1024 --steps 5e6"""
    import argparse
    import json

    from .tasks import make_task

    ap = argparse.ArgumentParser(prog="python -m paper_2410_00425_b200.learn")
    ap.add_argument("--task", default="CartpoleBalance")
    ap.add_argument("--envs", type=int, default=1024)
    ap.add_argument("--eval-envs", type=int, default=256)
    ap.add_argument("--steps", type=float, default=5e6)
    ap.add_argument("--rollout", type=int, default=32)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--time-limit", type=float, default=None)
    ap.add_argument("--target-success", type=float, default=None)
    ap.add_argument("--out", default=None)
    a = ap.parse_args(argv)
    cfg = PPOConfig(num_envs=a.envs, rollout_len=a.rollout, total_steps=int(a.steps), eval_envs=a.eval_envs)
    env = make_task(a.task, a.envs, seed=a.seed)
    ev = make_task(a.task, a.eval_envs, seed=a.seed + 1)
    net, rms, log = ppo_train(env, cfg, a.seed, ev, a.time_limit, log_fn=lambda r: print(json.dumps(r), flush=True),
                              target_success=a.target_success)
    summary = {"task": a.task, "env_steps": log.env_steps, "rollout_seconds": log.rollout_seconds,
               "update_seconds": log.update_seconds, "evals": log.evals, "config": cfg.__dict__}
    if a.out:
        with open(a.out, "w") as f:
            json.dump(summary, f, indent=1)
    print(json.dumps({k: v for k, v in summary.items() if k != "evals"}))
    return 0


if __name__ == "__main__":
    import sys

    sys.exit(main())
