"""TEST INFRASTRUCTURE: generates tests/golden/*.npz from the UNMODIFIED reference build
(oracle/_ref/libpbrl_ref.so).  The reference publishes no stored golden vectors (SURVEY.md
§8(c)), so these fixtures are the reference's own outputs on fixed seeds; they let the oracle be
pinned on a machine without /root/reference.

    python oracle/make_golden.py        # rewrites tests/golden/
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from oracle.oracle import Ref, sac_defaults, td3_defaults  # noqa: E402

OUT = ROOT / "tests" / "golden"
TD3_NETS = ("policy", "policy_target", "critic1", "critic2", "critic1_target", "critic2_target")
SAC_NETS = ("policy", "critic1", "critic2", "critic1_target", "critic2_target")


def td3_case(ref: Ref, name, n, ds, da, hidden, B, K, seed, bseed, bound=1.0, hyper=None):
    st = ref.td3(n, ds, da, hidden, bound, seed)
    hy = td3_defaults(n)
    hy.update(hyper or {})
    raw = ref.synthetic_batches(K, n, B, ds, da, bseed)
    init = {f"init_{k}": st.get_net(k) for k in TD3_NETS}
    losses = []
    for k in range(K):
        losses.append(st.step(tuple(x[k] for x in raw), hy, want_losses=True))
    out = dict(n=n, ds=ds, da=da, hidden=np.asarray(hidden), B=B, K=K, seed=seed, bseed=bseed,
               bound=bound, losses=np.asarray(losses), **init)
    for f, v in hy.items():
        out[f"hyper_{f}"] = np.asarray(v, np.float64)
    for k in TD3_NETS:
        out[f"final_{k}"] = st.get_net(k)
    for k in ("policy", "critic1", "critic2"):
        m, v, t = zip(*[st.get_adam(k, i) for i in range(n)])
        out[f"adam_m_{k}"], out[f"adam_v_{k}"], out[f"adam_t_{k}"] = np.stack(m), np.stack(v), np.asarray(t)
    out["delay_acc"], out["steps"] = st.counters()
    np.savez_compressed(OUT / f"{name}.npz", **out)


def sac_case(ref: Ref, name, n, ds, da, hidden, B, K, seed, bseed):
    st = ref.sac(n, ds, da, hidden, 1.0, seed)
    hy = sac_defaults(n, da)
    raw = ref.synthetic_batches(K, n, B, ds, da, bseed)
    for k in range(K):
        st.step(tuple(x[k] for x in raw), hy)
    out = dict(n=n, ds=ds, da=da, hidden=np.asarray(hidden), B=B, K=K, seed=seed, bseed=bseed)
    for k in SAC_NETS:
        out[f"final_{k}"] = st.get_net(k)
    la, am, av, at, steps = st.counters()
    out.update(log_alpha=la, alpha_m=am, alpha_v=av, alpha_t=at, steps=steps)
    np.savez_compressed(OUT / f"{name}.npz", **out)


def rng_case(ref: Ref):
    keys, uni, nrm = [], [], []
    for seed, stream, use, step in [(0, 0, 1, 0), (7, 3, 4, 99), (2**63 + 5, 12345, 12, 2**40),
                                    (1, 2, 8, 0)]:
        k = ref.stream_key(seed, stream, use, step)
        keys.append([seed, stream, use, step, k])
        uni.append([ref.uniform(k, c) for c in range(16)])
        nrm.append([ref.normal_pair(k, 2 * c) for c in range(16)])
    np.savez_compressed(OUT / "rng.npz", keys=np.asarray(keys, np.uint64), uniform=np.asarray(uni),
                        normal=np.asarray(nrm))


def replay_case(ref: Ref):
    n, ds, da, cap, B = 3, 4, 2, 50, 37
    rng = np.random.default_rng(5)
    bufs, pushed = [], []
    for m in range(n):
        rb = ref.replay(cap, ds, da)
        for i in range(30 + 25 * m):
            t = (rng.standard_normal(ds).astype(np.float32), rng.standard_normal(da).astype(np.float32),
                 np.float32(rng.standard_normal()), rng.standard_normal(ds).astype(np.float32),
                 np.float32(i % 5 == 0))
            rb.push(*t, member=m)
            pushed.append((m,) + t)
        bufs.append(rb)
    out = {"member": np.asarray([p[0] for p in pushed], np.uint32),
           "s": np.stack([p[1] for p in pushed]), "a": np.stack([p[2] for p in pushed]),
           "r": np.asarray([p[3] for p in pushed], np.float32), "s2": np.stack([p[4] for p in pushed]),
           "d": np.asarray([p[5] for p in pushed], np.float32), "cap": cap, "B": B}
    for draw in (0, 3):
        s, a, r, s2, d = ref.sample_batch(bufs, B, 0, n, 77, [0, 1, 2], draw)
        out.update({f"draw{draw}_s": s, f"draw{draw}_a": a, f"draw{draw}_r": r,
                    f"draw{draw}_s2": s2, f"draw{draw}_d": d})
    np.savez_compressed(OUT / "replay.npz", **out)


def pbt_case(ref: Ref):
    rng = np.random.default_rng(11)
    out = {}
    for n in (4, 10, 33, 80):
        rings = rng.standard_normal((n, 10)).round(1)
        counts = rng.integers(1, 11, n).astype(np.uint32)
        key = ref.stream_key(1, 0, 8, 0)
        rep, don, nxt = ref.pbt_plan(rings, counts, 0.3, key, 7)
        out.update({f"n{n}_rings": rings, f"n{n}_counts": counts, f"n{n}_order": ref.pbt_rank(rings, counts),
                    f"n{n}_replaced": rep, f"n{n}_donors": don, f"n{n}_next": np.uint64(nxt),
                    f"n{n}_key": np.uint64(key)})
    np.savez_compressed(OUT / "pbt.npz", **out)


def tanh_case(ref: Ref):
    rng = np.random.default_rng(3)
    x = np.concatenate([rng.standard_normal(4000).astype(np.float32) * 4,
                        np.float32([0.0, -0.0, 1e-30, -1e-8, 0.5, 22.0, -22.5, 9.0])])
    np.savez_compressed(OUT / "tanhf.npz", x=x, y=np.asarray([ref.tanhf(float(v)) for v in x], np.float32))


def act_case(ref: Ref):
    """act / sac_act (algos.hpp:895-942) on fixed observations, stochastic and deterministic."""
    out = {}
    obs = np.random.default_rng(5).uniform(-1, 1, (3, 4, 17)).astype(np.float32)
    steps = np.asarray([3, 0, 11], np.uint64)
    noise = np.asarray([0.1, 0.0, 0.3])
    out.update(obs=obs, steps=steps, noise=noise, seed=99, hidden=np.asarray([32, 32]), n=3,
               ds=17, da=6, state_seed=7)
    for algo in ("td3", "sac"):
        st = (ref.td3 if algo == "td3" else ref.sac)(3, 17, 6, [32, 32], 1.0, 7)
        for det in (0, 1):
            out[f"{algo}_det{det}"] = st.act(obs, 99, steps, noise, bool(det))
    np.savez_compressed(OUT / "act.npz", **out)


def f4_case(ref: Ref):
    """shared-critic TD3 with member masks and the DvD hook, shared-critic SAC, dvd_loss,
    median_pairwise_distance and CEM sample / update"""
    n, ds, da, hidden, B, K = 4, 5, 2, [8, 8], 6, 4
    out = dict(n=n, ds=ds, da=da, hidden=np.asarray(hidden), B=B, K=K)
    raw = ref.synthetic_batches(K, n, B, ds, da, 34)
    probe = np.random.default_rng(5).uniform(-1, 1, (n + 2, ds))
    out["probe"] = probe
    st = ref.td3(n, ds, da, hidden, 1.0, 33, shared=True)
    hy = td3_defaults(n)
    for k in range(K):
        dvd = {"probe": probe, "length_scale": 0.7, "jitter": 1e-6, "lam_start": 0.1,
               "lam_end": 0.7, "horizon": 4, "step": k}
        mask = [1, 1, 0, 0] if k == 1 else None
        if k == 3:
            st.step(tuple(x[k] for x in raw), hy, policy_mask=mask)
        else:
            st.step(tuple(x[k] for x in raw), hy, policy_mask=mask, dvd=dvd)
    for k in TD3_NETS:
        out[f"td3_{k}"] = st.get_net(k)
    ss = ref.sac(n, ds, da, hidden, 1.0, 41, shared=True)
    for k in range(K):
        ss.step(tuple(x[k] for x in raw), sac_defaults(n, da))
    for k in SAC_NETS:
        out[f"sac_{k}"] = ss.get_net(k)
    rng = np.random.default_rng(9)
    e = rng.normal(size=(7, 12))
    out["dvd_emb"] = e
    loss, logdet, grad = ref.dvd_loss(e, 0.9, 1e-8, 1.3)
    out["dvd_loss"], out["dvd_logdet"], out["dvd_grad"] = loss, logdet, grad
    out["median"] = ref.median_pairwise_distance(e)
    mean, var = rng.normal(size=37), rng.uniform(0, 0.1, 37)
    key = ref.stream_key(7, 2, 10, 0)
    cand, nxt = ref.cem_sample(mean, var, 1e-2, 6, key, 4)
    scores = rng.normal(size=6)
    m2, v2, nz = ref.cem_update(mean, var, 1e-2, cand, scores)
    out.update(cem_mean=mean, cem_var=var, cem_key=np.uint64(key), cem_cand=cand,
               cem_next=np.uint64(nxt), cem_scores=scores, cem_mean2=m2, cem_var2=v2,
               cem_noise2=nz)
    np.savez_compressed(OUT / "f4.npz", **out)


def main():
    ref = Ref()
    OUT.mkdir(parents=True, exist_ok=True)
    if sys.argv[1:] == ["act"]:
        act_case(ref)
        return
    if sys.argv[1:] == ["f4"]:
        f4_case(ref)
        return
    td3_case(ref, "td3_small", 3, 4, 2, [8, 8], 8, 20, 11, 12,
             hyper=dict(policy_delay_ratio=[0.5, 1.0, 0.3], critic_lr=[3e-4, 1e-3, 3e-4]))
    td3_case(ref, "td3_halfcheetah", 2, 17, 6, [64, 64], 32, 4, 7, 7)
    sac_case(ref, "sac_small", 3, 4, 2, [8, 8], 8, 10, 21, 22)
    rng_case(ref)
    replay_case(ref)
    pbt_case(ref)
    tanh_case(ref)
    act_case(ref)
    f4_case(ref)
    print("golden fixtures written to", OUT)


if __name__ == "__main__":
    main()
