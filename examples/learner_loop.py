"""The run_training learner loop (pipeline_run.hpp:77-468) driven through the B200 path: a
population of TD3 agents on a vectorised PointMass (a numpy restatement of envs.cpp:73-110, the
reference's desk environment), with every per-step piece of the hot path on the device:

  actors   act()                     (algos.hpp:895-915)      -> pbrl_act
  ingest   ReplayBuffer::push        (replay.hpp:56-69)       -> pbrl_replay_insert (batched)
  learner  sample_batch + update_k   (pipeline_run.hpp:230-355) -> pbrl_update_k
  PBT      pbt_evolve_trainer        (evolve.hpp:169-190)     -> device rank / copies / resets
  export   save_checkpoint           (net_pop.hpp:245-261)    -> pbrl_save_checkpoint

The reference runs actors, ingest, prefetch and learner as threads with a ratio controller; this
demo interleaves them on one thread (the update-to-data ratio is fixed by --updates-per-step).

    python examples/learner_loop.py [--pop 16 --envs 8 --iters 60 --precision bf16]
"""
from __future__ import annotations

import argparse
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import paper_2206_08888_b200 as pb  # noqa: E402

ARENA, MAX_SPEED, DT, HORIZON = 1.0, 1.0, 0.05, 100  # envs.cpp constants for PointMass


class PointMass:
    """Vectorised PointMass (envs.cpp:61-110): obs (px, py, vx, vy), action (ax, ay) in
    [-1, 1], reward = -|p|, episodes of HORIZON steps; shape [pop, envs]."""

    def __init__(self, pop, envs, seed):
        self.rng = np.random.default_rng(seed)
        self.shape = (pop, envs)
        self.reset(np.ones(self.shape, bool))

    def reset(self, mask):
        n = int(mask.sum())
        if not hasattr(self, "phys"):
            self.phys = np.zeros(self.shape + (4,))
            self.t = np.zeros(self.shape, int)
            self.ret = np.zeros(self.shape)
        self.phys[mask] = np.concatenate([self.rng.uniform(-0.5, 0.5, (n, 2)), np.zeros((n, 2))], 1)
        self.t[mask] = 0
        self.ret[mask] = 0.0

    def step(self, a):
        a = np.clip(a, -1.0, 1.0)
        p, v = self.phys[..., :2], self.phys[..., 2:]
        nxt = p + v * DT
        pc = np.clip(nxt, -ARENA, ARENA)
        v = np.where(nxt != pc, 0.0, v)  # walls absorb the normal velocity component
        v = np.clip(v + a * DT, -MAX_SPEED, MAX_SPEED)
        self.phys = np.concatenate([pc, v], -1)
        r = -np.sqrt((pc ** 2).sum(-1))
        self.t += 1
        self.ret += r
        return self.phys.copy(), r, self.t >= HORIZON


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--pop", type=int, default=16)
    ap.add_argument("--envs", type=int, default=8)
    ap.add_argument("--iters", type=int, default=60)
    ap.add_argument("--updates-per-step", type=int, default=1)
    ap.add_argument("--batch", type=int, default=256)
    ap.add_argument("--precision", default="bf16")
    ap.add_argument("--pbt-interval", type=int, default=20)
    ap.add_argument("--out", default=None, help="checkpoint of the final policies")
    args = ap.parse_args()

    n, E, seed = args.pop, args.envs, 7
    st = pb.make_td3_state(n, 4, 2, [256, 256], 1.0, seed, precision=args.precision)
    rng = pb.RngSequence(seed, 0, "kHyperDraw", 0)  # as run_training (pipeline_run.hpp:116)
    prior = pb.Td3Prior()
    hy = pb.Td3Hyper.defaults(n)
    for m in range(n):
        hy.set_member(m, prior.sample_member(rng))
    replay = pb.DeviceReplay(st, 100_000, "per_agent")
    pbt = pb.PBTState(n)
    pbt_rng = pb.RngSequence(seed, 0, "kDonorChoice", 0)  # pipeline_run.hpp:140
    env = PointMass(n, E, seed)
    steps = np.zeros(n, np.uint64)
    draw, t0, events = 0, time.perf_counter(), 0
    for it in range(args.iters):
        for _ in range(HORIZON // 4):
            obs = env.phys.astype(np.float32)
            act = pb.act(st, obs, hy.explore_std, seed, steps)  # [n, E, 2]
            steps += 1
            obs2, r, done = env.step(act)
            mem = np.repeat(np.arange(n, dtype=np.uint32), E)
            replay.insert(obs.reshape(-1, 4), act.reshape(-1, 2), r.reshape(-1),
                          obs2.reshape(-1, 4).astype(np.float32),
                          done.reshape(-1).astype(np.float32), mem)
            if done.any():
                for m, e in zip(*np.nonzero(done)):
                    pbt.record_return(int(m), float(env.ret[m, e]))
                env.reset(done)
            k = args.updates_per_step
            if pb.update_k_from_replay(st, replay, k, hy, args.batch, seed, draw, min_size=1000):
                draw += k
        if (it + 1) % args.pbt_interval == 0 and pbt.every_member_scored():
            plan = pb.pbt_evolve_trainer(pbt, st, hy, prior, pbt_rng)
            if plan is not None:
                events += 1
                print(f"iter {it + 1}: PBT replaced {list(plan.replaced)} from "
                      f"{list(plan.donors)}")
        if (it + 1) % 10 == 0 and pbt.every_member_scored():
            f = pbt.fitness()
            print(f"iter {it + 1:4d}: updates {draw:6d}  mean return {f.mean():8.2f}  "
                  f"best {f.max():8.2f}  ({time.perf_counter() - t0:.1f} s)")
    if args.out:
        pb.save_checkpoint(st, "policy", args.out)
        print("policy checkpoint (PBRLNET1):", args.out)
    print(f"done: {draw} update steps x {n} members, {events} PBT events")


if __name__ == "__main__":
    main()
