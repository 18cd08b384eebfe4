#!/usr/bin/env python
"""Population TD3 update throughput on B200 (BASELINE.json metric: population agent-updates/s,
TD3 pop=80, MLP 2x256, batch 256, obs 17 / act 6).

One "step" = one td3_update_step of the whole population over one synthetic batch
(make_synthetic_batches semantics, bench.hpp:69-93) -- exactly what the reference's
bench_update times per step (bench.hpp:116-118).  Under torchrun the population is sharded in
contiguous member blocks (80/N per GPU, RNG streams keyed by global member id), no per-step
collective; the max over ranks of the device time is reported.

    python bench.py [--gpus N --steps K --warmup W] [--impl reference] [--precision P]

Prints ONE JSON line (rank 0).  `value` = agent-updates/s with inputs resident in HBM (CUDA
events on the library's stream); `e2e` = the same through the C ABI with pinned HOST batches
(H2D of each step's batch and D2H of its losses inside the timed region).
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

CONFIGS = {
    # name: algo, total population, hidden, batch  (BASELINE.json configs)
    "A": dict(algo="td3", pop=4, hidden=[256, 256], batch=256),
    "B": dict(algo="td3", pop=10, hidden=[256, 256], batch=256),
    "C": dict(algo="sac", pop=32, hidden=[256, 256], batch=256),
    "D": dict(algo="td3", pop=80, hidden=[256, 256], batch=256),
    "E": dict(algo="td3", pop=256, hidden=[512, 512, 512], batch=1024),
}
OBS, ACT, SEED = 17, 6, 7
L2_BYTES = 126 * 2 ** 20
METRIC = "population agent-updates/sec (TD3, pop=80) at 1/2/4/8 B200; % of roofline"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="D", choices=sorted(CONFIGS))
    ap.add_argument("--pop", type=int, default=None, help="override the total population")
    ap.add_argument("--precision", default=os.environ.get("PBRL_PRECISION", "bf16"),
                    choices=["ffma32", "bf16", "tf32"])
    ap.add_argument("--scaling", default="strong", choices=["weak", "strong"],
                    help="strong (default, BASELINE config D: pop 80 sharded over N GPUs): the "
                         "config's population split over the N ranks; weak: every rank runs the "
                         "config's population (members keyed by global id, total = pop x N)")
    ap.add_argument("--memory-budget-gib", type=float, default=None,
                    help="bench_update's memory budget (bench.hpp:35,141-147): ResourceError when "
                         "the estimated device footprint exceeds it (default: free HBM)")
    ap.add_argument("--pbt-interval", type=int, default=1000,
                    help="updates between PBT exchanges; one exchange (fitness all-gather, device "
                         "plan, exploit copies, resets) is timed and amortised over it")
    ap.add_argument("--pbt-timeout", type=float, default=180.0,
                    help="seconds the timed PBT exchange may take before the line is printed "
                         "without it")
    ap.add_argument("--reps", type=int, default=5,
                    help="the K timed steps are split into this many equal repetitions for the "
                         "median / IQR (bench.hpp:184-200)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--replay", action="store_true",
                    help="replay-inclusive variant (SURVEY.md §8(d)): per-agent HBM rings "
                         "pre-filled with 100,000 synthetic transitions per member, every step "
                         "samples its batch on the device (draw_id = step, min_size 1000)")
    ap.add_argument("--profile-json", default=None, help="write the per-class profile here")
    return ap.parse_args()


def peaks(precision="bf16"):
    """Roofline denominators: HBM GB/s and the dense tensor peak of the arithmetic the kernels
    use -- bf16 from the driver-written MEASURED_PEAKS.json; TF32 (which that file lacks) from
    profiles/measured_tf32.json (tools/measure_tf32_peak.py, same method), else half of bf16."""
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        pk = dict(hbm=d["hbm_gbs"], tensor=d.get("bf16_tflops_sustained", d["bf16_tflops"]),
                  tensor_burst=d["bf16_tflops"], src="measured (MEASURED_PEAKS.json)")
    else:
        pk = dict(hbm=6650.0, tensor=1400.0, tensor_burst=1590.0,
                  src="fallback (B200_PROFILING.md)")
    if precision == "tf32":
        t = ROOT / "profiles" / "measured_tf32.json"
        if t.exists():
            d = json.loads(t.read_text())
            pk.update(tensor=d["tf32_tflops_sustained"], tensor_burst=d["tf32_tflops"])
            pk["src"] += "; tf32 measured (profiles/measured_tf32.json)"
        else:
            pk.update(tensor=pk["tensor"] / 2, tensor_burst=pk["tensor_burst"] / 2)
            pk["src"] += "; tf32 = bf16 / 2 (nominal ratio)"
    return pk


def td3_member_update_work(hidden, batch, f=0.5, ds=OBS, da=ACT):
    """minimal FLOP and compulsory HBM bytes of one TD3 member-update (policy
    fires every 1/f steps): MACs/row = F_P + 2F_C + 2(3F_C - F_C1)
    + f(2F_P + (F_P - F_P1) + 2F_C - F_C1 + da H1); bytes = 28(2P_C + f P_P) + 8f(P_P + 2P_C)
    (fused Adam + Polyak, fp32) + 2 B 42 4 (replay gather read + write)."""
    pd, cd = [ds] + list(hidden) + [da], [ds + da] + list(hidden) + [1]
    F = lambda d: sum(d[i] * d[i + 1] for i in range(len(d) - 1))
    P = lambda d: sum(d[i] * d[i + 1] + d[i + 1] for i in range(len(d) - 1))
    FP, FC, FP1, FC1, H1 = F(pd), F(cd), pd[0] * pd[1], cd[0] * cd[1], hidden[0]
    macs = FP + 2 * FC + 2 * (3 * FC - FC1) + f * (2 * FP + (FP - FP1) + 2 * FC - FC1 + da * H1)
    PP, PC = P(pd), P(cd)
    byt = 28 * (2 * PC + f * PP) + 8 * f * (PP + 2 * PC) + 2 * batch * (2 * ds + da + 2) * 4
    return 2.0 * batch * macs, float(byt)


def sac_member_update_work(hidden, batch, ds=OBS, da=ACT):
    """The same minimal FLOP / compulsory-byte model for one SAC member-update (the policy and
    the temperature update every step, sac_update_step algos.hpp:782-835; Gaussian policy head of
    2·da outputs, twin critics with Polyak targets, no target policy): MACs/row =
    (F_P + 2F_C) target + 2F_C + 2(2F_C - F_C1) critics + F_P + 2F_C + 2(F_C - F_C1 + da H1)
    + (2F_P - F_P1) policy; bytes = 28(2P_C + P_P) + 8(2P_C) + 2 B 42 4."""
    pd, cd = [ds] + list(hidden) + [2 * da], [ds + da] + list(hidden) + [1]
    F = lambda d: sum(d[i] * d[i + 1] for i in range(len(d) - 1))
    P = lambda d: sum(d[i] * d[i + 1] + d[i + 1] for i in range(len(d) - 1))
    FP, FC, FP1, FC1, H1 = F(pd), F(cd), pd[0] * pd[1], cd[0] * cd[1], hidden[0]
    macs = (FP + 2 * FC) + 2 * FC + 2 * (2 * FC - FC1) + FP + 2 * FC \
        + 2 * (FC - FC1 + da * H1) + (2 * FP - FP1)
    PP, PC = P(pd), P(cd)
    byt = 28 * (2 * PC + PP) + 8 * (2 * PC) + 2 * batch * (2 * ds + da + 2) * 4
    return 2.0 * batch * macs, float(byt)


# ------------------------------------------------------------------ clocks during the timed region
class Clocks:
    """Samples SM clock and throttle reasons through NVML every 1 ms while the timed region
    runs (the recipe's nvidia-smi clocks line, at a rate that resolves sub-second regions)."""

    REASONS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
               "sw_power_cap": 0x4, "hw_power_brake_slowdown": 0x80}

    def __init__(self, gpu: int):
        self.gpu, self.rows, self.stop = gpu, [], threading.Event()

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            idx = int(vis.split(",")[self.gpu]) if vis else self.gpu
            self.h = pynvml.nvmlDeviceGetHandleByIndex(idx)
            self.nv = pynvml
            self.max = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.t = threading.Thread(target=self._loop, daemon=True)
            self.t.start()
        except Exception as e:  # pragma: no cover - no NVML
            self.nv, self.err = None, str(e)
        return self

    def _loop(self):
        nv = self.nv
        while not self.stop.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                self.rows.append((sm, rs))
            except Exception:
                pass
            time.sleep(0.001)

    def __exit__(self, *a):
        self.stop.set()
        if self.nv:
            self.t.join(timeout=2)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"], "samples": 0}
        sm = sorted(r[0] for r in self.rows)
        reasons = sorted({k for _, rs in self.rows for k, bit in self.REASONS.items() if rs & bit})
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": self.max, "reasons": reasons,
                "samples": len(self.rows), "source": "nvml 1 ms"}


# ------------------------------------------------------------------ CPU baseline (reference build)
def cpu_reference(cfg, pop, k_steps=2, reps=3):
    """Reference bench_update<float> vectorized (bench.hpp:137-227) on the host cores."""
    from oracle.oracle import load_ref
    ref = load_ref()
    cores = os.cpu_count()
    if ref is not None:
        r = ref.bench_update(1, 0 if cfg["algo"] == "td3" else 1, pop, k_steps, reps,
                             cfg["batch"], cfg["hidden"], budget=64 << 30)
        v = pop * k_steps / (r["median_ms"] / 1e3)
        return dict(value=v, unit="agent-updates/s", cores=cores, kind="reference",
                    sample=f"reference bench_update<float> vectorized, pop {pop}, "
                           f"{'x'.join(map(str, cfg['hidden']))} MLP, batch {cfg['batch']}, "
                           f"k={k_steps} steps x {reps} reps (median), ThreadPool "
                           f"{cores - 1} workers + caller")
    # the reference could not be built on this host: the C restatement, single thread
    from oracle.oracle import load_oracle, td3_defaults, sac_defaults
    ora = load_oracle()
    st = (ora.td3 if cfg["algo"] == "td3" else ora.sac)(pop, OBS, ACT, cfg["hidden"], 1.0, SEED)
    hy = td3_defaults(pop) if cfg["algo"] == "td3" else sac_defaults(pop, ACT)
    raw = ora.synthetic_batches(k_steps, pop, cfg["batch"], OBS, ACT, SEED)
    t0 = time.perf_counter()
    for k in range(k_steps):
        st.step(tuple(x[k] for x in raw), hy)
    dt = time.perf_counter() - t0
    return dict(value=pop * k_steps / dt, unit="agent-updates/s", cores=1, kind="port",
                sample=f"C restatement oracle, pop {pop}, k={k_steps} steps, one thread")


def reference_arm(args, cfg, pop, rank, world):
    if rank != 0:
        return
    k = 2 if args.steps >= 2 else 1
    gpus = max(world, args.gpus)
    total = pop * gpus if args.scaling == "weak" else pop  # the same workload as our arm
    cb = cpu_reference(cfg, total, k_steps=k, reps=3)
    line = {"impl": "reference", "metric": METRIC, "value": cb["value"], "unit": cb["unit"],
            "n_gpus": gpus, "steps": k, "warmup": 1, "ms_per_step": total / cb["value"] * 1e3,
            "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None,
            "dtype": "f32", "data": "synthetic (make_synthetic_batches, seed 7)",
            "config": config_dict(args, cfg, total, "host", gpus),
            "cpu_baseline": cb,
            "e2e": {"value": cb["value"], "unit": cb["unit"], "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def config_dict(args, cfg, pop, l2, gpus):
    per = pop // max(1, gpus)
    return {"workload": f"{cfg['algo'].upper()} population update, config {args.config}: "
                        f"pop {per} per GPU ({pop} total), MLP "
                        f"{'x'.join(map(str, cfg['hidden']))}, batch {cfg['batch']}, "
                        f"obs {OBS} / act {ACT}",
            "algo": cfg["algo"], "population": pop, "population_per_gpu": per,
            "hidden": cfg["hidden"], "batch": cfg["batch"], "obs_dim": OBS, "act_dim": ACT,
            "parallelism": f"population shards x{gpus} ({args.scaling} scaling, no per-step "
                           f"collective)", "precision": args.precision, "l2": l2,
            "inputs": "device replay rings (sampled per step)" if getattr(args, "replay", False)
                      else "50 synthetic batches resident in HBM"}


# ------------------------------------------------------------------ our arm
def spawn_ranks(args):
    """`--gpus N` without a launcher: re-run this script under torch.distributed.run with N
    ranks (one per GPU, rendezvous on 127.0.0.1); rank 0's JSON line is passed through."""
    import socket
    import subprocess
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1", "--master-port",
           str(port), str(Path(__file__).resolve())] + sys.argv[1:]
    return subprocess.run(cmd).returncode


def estimated_bytes(cfg, n, nb, precision):
    """bench_estimated_bytes (bench.cpp:37-56) for the device layout: per member the fp32
    parameters, targets, Adam moments and gradients of every network (+ bf16 operand copies),
    the nb resident synthetic batches, and the activation scratch of one step."""
    hid = cfg["hidden"]
    pd, cd = [OBS] + hid + [ACT], [OBS + ACT + 1] + hid + [1]
    P = lambda d: sum(d[i] * d[i + 1] + d[i + 1] for i in range(len(d) - 1))
    PP = P(pd) + (P(pd) if cfg["algo"] == "sac" else 0)
    per_param = 5 * 4 + (4 if precision == "bf16" else 0)
    state = n * (PP + 2 * P(cd)) * per_param
    batches = nb * n * cfg["batch"] * (2 * OBS + ACT + 2) * 4
    scratch = n * cfg["batch"] * sum(hid) * 4 * 12
    return state + batches + scratch


def main():
    args = parse()
    cfg = dict(CONFIGS[args.config])
    pop = args.pop or cfg["pop"]
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        raise SystemExit(spawn_ranks(args))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        reference_arm(args, cfg, pop, rank, world)
        return

    import torch
    import torch.distributed as dist
    ndev = max(1, torch.cuda.device_count())
    # one rank per GPU over NCCL; with fewer GPUs than ranks (tests, or PBRL_BENCH_BACKEND=gloo)
    # the ranks share devices round-robin and the collectives run on the host (gloo)
    backend = os.environ.get("PBRL_BENCH_BACKEND", "nccl" if world <= ndev else "gloo")
    gpu = local % ndev
    torch.cuda.set_device(gpu)
    dev = torch.device("cuda", gpu)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    import paper_2206_08888_b200 as pb
    from paper_2206_08888_b200 import _lib
    from paper_2206_08888_b200.errors import ResourceError

    if args.scaling == "weak":  # every rank: the config's population, global member ids
        n = pop
        pop = pop * world
    else:
        if pop % world:
            raise SystemExit(f"population {pop} does not split over {world} GPUs")
        n = pop // world
    off = rank * n
    nb = 50  # bench_update's k = 50 distinct batches (bench.hpp:151), resident in HBM
    need = estimated_bytes(cfg, n, nb, args.precision)
    budget = (args.memory_budget_gib * 2 ** 30 if args.memory_budget_gib
              else torch.cuda.mem_get_info(dev)[0])
    if need > budget:
        raise ResourceError(f"bench_update: population of {n} needs an estimated {need} bytes, "
                            f"over the budget of {int(budget)}")
    make = pb.make_td3_state if cfg["algo"] == "td3" else pb.make_sac_state
    st = make(n, OBS, ACT, cfg["hidden"], 1.0, SEED, precision=args.precision, device=gpu,
              member_offset=off, n_global=pop)
    hy = pb.Td3Hyper.defaults(n) if cfg["algo"] == "td3" else pb.SacHyper.defaults(n, ACT)
    st._sync_hyper(hy)

    # synthetic inputs in HBM: 50 distinct global batches (bench_update's k=50), local slice
    gb = pb.make_synthetic_batches(nb, pop, cfg["batch"], OBS, ACT, SEED, device=dev)
    batches = [pb.TransitionBatch(*[x[off:off + n].contiguous() for x in
                                    (b.s, b.a, b.r, b.s2, b.done)]) for b in gb]
    del gb
    B = cfg["batch"]

    def make_runner(p, bl):
        structs = [_lib.Batch(*[x.data_ptr() for x in (b.s, b.a, b.r, b.s2, b.done)])
                   for b in bl]

        def run(i, cnt=1):
            # cnt consecutive steps in one call (update_k_steps over a list of batches): inside
            # a call the pack of batch i+1 overlaps step i's last Adam
            arr = (_lib.Batch * cnt)(*[structs[(i + j) % len(structs)] for j in range(cnt)])
            _lib.call("pbrl_update_batches_device", p.handle, arr, cnt, B, None)
        return run

    run = make_runner(st, batches)
    replay_note = None
    if args.replay:
        # replay-inclusive: the device rings of run_training's learner (sample_batch +
        # update_k_steps fused, pbrl_update_k), filled with U[-1, 1) transitions, done ~ 0.02
        import numpy as np
        cap, chunk = 100_000, 5_000
        rb = pb.DeviceReplay(st, cap, "per_agent")
        rng = np.random.default_rng(SEED + rank)
        for c0 in range(0, cap, chunk):
            rows = n * chunk
            s_ = rng.uniform(-1, 1, (rows, OBS)).astype(np.float32)
            a_ = rng.uniform(-1, 1, (rows, ACT)).astype(np.float32)
            r_ = rng.uniform(-1, 1, rows).astype(np.float32)
            s2_ = rng.uniform(-1, 1, (rows, OBS)).astype(np.float32)
            d_ = (rng.uniform(0, 1, rows) < 0.02).astype(np.float32)
            rb.insert(s_, a_, r_, s2_, d_, np.repeat(np.arange(n, dtype=np.uint32), chunk))
        ready = C.c_int()

        def run(i, cnt=1):
            for j in range(cnt):
                _lib.call("pbrl_update_k", st.handle, 1, SEED, i + j, B, 1000, C.byref(ready))
                if not ready.value:
                    raise RuntimeError("replay rings not ready")
        replay_note = (f"per-agent HBM rings, {cap} transitions per member, min_size 1000, "
                       "draw_id = step (pbrl_update_k: device sample_batch + update)")
        args.no_e2e = True
    lstream = st.lib_stream()

    state_bytes = st.device_bytes()
    in_bytes = sum(x.numel() * 4 for b in batches for x in (b.s, b.a, b.r, b.s2, b.done))
    flush = (state_bytes + in_bytes) < 2 * L2_BYTES
    flush_buf = torch.empty(2 * L2_BYTES // 4, dtype=torch.float32, device=dev) if flush else None

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev if backend == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    for i in range(args.warmup):
        run(i)
    st.synchronize()

    # ---- timed region: K steps, device time on the library stream, max over ranks.  The K
    # steps are recorded as `reps` equal repetitions (bench.hpp:184-200: median / IQR).
    K = args.steps
    R = max(1, min(args.reps, K))
    edges = [round(K * j / R) for j in range(R + 1)]
    launches0 = st.launch_count()
    with Clocks(gpu) as clk:
        barrier()
        torch.cuda.synchronize(dev)
        st.synchronize()
        step_ms = []
        if not flush:
            evs = [torch.cuda.Event(enable_timing=True) for _ in range(R + 1)]
            evs[0].record(lstream)
            for j in range(R):
                # the rep's steps in calls of up to 50 batches (bench_update's k = 50)
                for i in range(edges[j], edges[j + 1], nb):
                    run(args.warmup + i, min(nb, edges[j + 1] - i))
                evs[j + 1].record(lstream)
            evs[-1].synchronize()
            rep_ms = [evs[j].elapsed_time(evs[j + 1]) for j in range(R)]
            total_ms = sum(rep_ms)
        else:
            pairs = []
            for i in range(K):
                with torch.cuda.stream(lstream):
                    flush_buf.fill_(float(i))  # evict L2 between steps (outside the events)
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(lstream)
                run(args.warmup + i)
                b.record(lstream)
                pairs.append((a, b))
            st.synchronize()
            step_ms = [a.elapsed_time(b) for a, b in pairs]
            rep_ms = [sum(step_ms[edges[j]:edges[j + 1]]) for j in range(R)]
            total_ms = sum(step_ms)
        st.synchronize()
        torch.cuda.synchronize(dev)
        barrier()
    launches = st.launch_count() - launches0
    total_ms = max_over_ranks(total_ms)
    value = pop * K / (total_ms / 1e3)
    per_step = sorted(r / max(1, edges[j + 1] - edges[j]) for j, r in enumerate(rep_ms))

    def quantile(v, q):
        x = q * (len(v) - 1)
        lo = int(x)
        hi = min(lo + 1, len(v) - 1)
        return v[lo] + (v[hi] - v[lo]) * (x - lo)
    reps = {"n": R, "steps_per_rep": K // R, "median_ms_per_step": quantile(per_step, 0.5),
            "iqr_ms_per_step": quantile(per_step, 0.75) - quantile(per_step, 0.25),
            "note": "this rank's repetitions; value / ms_per_step use the max over ranks"}

    # ---- event-instrumented pass over the same workload: per-kernel-class roofline
    kp = min(K, 10) if K >= 2 else 1
    _lib.call("pbrl_profile_begin", st.handle)
    for i in range(kp):
        run(args.warmup + K + i)
    buf = C.create_string_buffer(1 << 16)
    _lib.call("pbrl_profile_end", st.handle, buf, len(buf))
    prof = json.loads(buf.value.decode())
    if args.profile_json and rank == 0:
        Path(args.profile_json).write_text(json.dumps(prof, indent=1))
    pk = peaks(args.precision)
    cls = prof["classes"]
    # the dominant kernel class among those with algorithmic work (the SAC heads and other
    # elementwise launches carry no FLOP / byte model of their own)
    worked = [c for c in cls if cls[c]["flops"] > 0 or cls[c]["bytes"] > 0] or list(cls)
    dom = max(worked, key=lambda c: cls[c]["ms"])
    dc = cls[dom]
    avg_ms = dc["ms"] / max(1, dc["launches"])
    # the kernel class's bound is whichever of its algorithmic FLOPs (at the tensor peak) and
    # algorithmic bytes (at the HBM peak) takes longer: with fp32 activations at these shapes
    # (256-row batches, 256-wide layers: ~43 FLOP/B) the grouped GEMMs sit below the ridge
    t_tc = dc["flops"] / (pk["tensor"] * 1e12)
    t_mem = dc["bytes"] / (pk["hbm"] * 1e9)
    if t_tc >= t_mem:
        achieved = dc["flops"] / (dc["ms"] / 1e3) / 1e12
        roof = {"bound": "tensor", "achieved": achieved, "peak": pk["tensor"], "unit": "TFLOP/s",
                "frac": achieved / pk["tensor"]}
    else:
        achieved = dc["bytes"] / (dc["ms"] / 1e3) / 1e9
        roof = {"bound": "hbm", "achieved": achieved, "peak": pk["hbm"], "unit": "GB/s",
                "frac": achieved / pk["hbm"]}
    roof["tensor_frac"] = (dc["flops"] / (dc["ms"] / 1e3) / 1e12) / pk["tensor"]
    tot_ms = sum(c["ms"] for c in cls.values())
    roof.update({"traffic": None, "kernel": dom, "kernel_share_of_step": dc["ms"] / tot_ms,
                 "avg_launch_ms": avg_ms, "peak_source": pk["src"],
                 "algorithmic_flops_per_launch": dc["flops"] / max(1, dc["launches"]),
                 "algorithmic_bytes_per_launch": dc["bytes"] / max(1, dc["launches"])})
    # HBM fraction of every byte-bound class (north_star: gather and Adam against HBM peak)
    classes_hbm = {k: {"gbs": c["bytes"] / (c["ms"] / 1e3) / 1e9 if c["ms"] > 0 else None,
                       "frac": (c["bytes"] / (c["ms"] / 1e3) / 1e9) / pk["hbm"]
                       if c["ms"] > 0 else None}
                   for k, c in cls.items()
                   if k in ("adam_polyak", "gather_pack", "elementwise") and c["bytes"] > 0}
    # whole-step roofline: T_roof = max(n F / P_tc, n Bytes / BW_hbm)
    work = td3_member_update_work if cfg["algo"] == "td3" else sac_member_update_work
    fl, by = work(cfg["hidden"], cfg["batch"])
    t_roof = max(n * fl / (pk["tensor"] * 1e12), n * by / (pk["hbm"] * 1e9))
    step_roof = {"flops_per_member_update": fl, "bytes_per_member_update": by,
                 "t_roof_ms_per_step": t_roof * 1e3,
                 "bound": "tensor" if n * fl / pk["tensor"] / 1e12 > n * by / pk["hbm"] / 1e9
                 else "hbm",
                 "frac": t_roof * 1e3 / (total_ms / K),
                 "roofline_agent_updates_per_s": pop / t_roof}
    tfile = ROOT / "profiles" / f"traffic_{args.precision}_{args.config}.json"
    if tfile.exists():
        try:
            roof["traffic"] = json.loads(tfile.read_text()).get(dom)
        except Exception:
            pass

    # ---- e2e through the C ABI: pinned host batches, every step's H2D copy and the D2H of every
    # step's losses inside the timed region.  update_k_steps semantics (algos.hpp:953-983): each
    # call runs KC = 50 host batches -- the reference bench's K --
    # with the copy of batch i+1 overlapping step i, and returns the KC steps' critic1 / critic2 /
    # policy losses.
    e2e = None
    if not args.no_e2e:
        hb = [[x.cpu().pin_memory() for x in (b.s, b.a, b.r, b.s2, b.done)] for b in batches[:10]]
        hstructs = [_lib.Batch(*[x.data_ptr() for x in h]) for h in hb]
        KC = 50
        loss = torch.empty(KC * 3 * n, dtype=torch.float64).pin_memory()
        lptr = C.cast(loss.data_ptr(), _lib.f64p)
        calls = max(1, min(K, 100) // KC)

        def run_host(c):
            arr = (_lib.Batch * KC)(*[hstructs[(c * KC + j) % len(hstructs)] for j in range(KC)])
            _lib.call("pbrl_update_batches_losses", st.handle, arr, KC, B, None, lptr)

        run_host(0)
        barrier()
        st.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record(lstream)
        for c in range(calls):
            run_host(c + 1)
        e1.record(lstream)
        e1.synchronize()
        wall = time.perf_counter() - t0
        ems = max_over_ranks(e0.elapsed_time(e1))
        ke = calls * KC
        e2e = {"value": pop * ke / (ems / 1e3), "unit": "agent-updates/s",
               "h2d_bytes_per_step": n * B * (2 * OBS + ACT + 2) * 4,
               "d2h_bytes_per_step": 3 * n * 8, "steps": ke, "steps_per_call": KC,
               "host_wall_value": pop * ke / wall}

    # ---- config B: vectorization overhead, t(pop 10) / t(pop 1) per step (target <= 1.5)
    vec = None
    if args.config == "B" and world == 1:
        one = make(1, OBS, ACT, cfg["hidden"], 1.0, SEED, precision=args.precision, device=gpu)
        one._sync_hyper(pb.Td3Hyper.defaults(1))
        b1 = [pb.TransitionBatch(*[x[:1].contiguous() for x in (b.s, b.a, b.r, b.s2, b.done)])
              for b in batches]
        run1 = make_runner(one, b1)
        for i in range(args.warmup):
            run1(i)
        one.synchronize()
        ls1 = one.lib_stream()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(ls1)
        for i in range(K):
            run1(args.warmup + i)
        e1.record(ls1)
        e1.synchronize()
        t1 = e0.elapsed_time(e1) / K
        vec = {"t_pop1_ms_per_step": t1, "t_pop10_ms_per_step": total_ms / K,
               "ratio": (total_ms / K) / t1, "target": 1.5}

    # ---- PBT exchange, timed separately: fitness all-gather over
    # the ranks, identical device plan, exploit copies (cross-rank member blobs over NCCL,
    # same-rank on device), optimiser resets and hyper re-draws; amortised over pbt_interval
    # updates.  Returns are synthetic: record_return from RngStream::of(7, m, kGeneric, event).
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_reference(cfg, pop)

    line = None
    if rank == 0:
        ngpu = min(world, ndev) if backend != "nccl" else world
        line = {"metric": METRIC, "value": value, "unit": "agent-updates/s", "n_gpus": ngpu,
                "steps": K, "warmup": args.warmup, "ms_per_step": total_ms / K,
                "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None,
                "dtype": {"ffma32": "f32", "bf16": "bf16", "tf32": "tf32"}[args.precision],
                "data": ("synthetic (make_synthetic_batches semantics, seed 7, 50 batches in HBM)"
                         if not replay_note else "synthetic transitions in device replay rings: "
                         + replay_note),
                "config": config_dict(args, cfg, pop,
                                      "flushed between steps" if flush else
                                      f"inputs+state {(state_bytes + in_bytes) / 2**20:.0f} MiB "
                                      f"per GPU > L2", world),
                "roofline": roof, "step_roofline": step_roof, "class_hbm": classes_hbm,
                "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches, "reps": reps,
                "pbt_exchange": None, "vectorization_overhead": vec,
                "ranks": world, "backend": backend if world > 1 else None,
                "clocks": clk.summary(), "profile": {k: {kk: round(vv, 6) if isinstance(vv, float)
                                                         else vv for kk, vv in v.items()}
                                                     for k, v in cls.items()}}
    # ---- PBT exchange (after the line is assembled): an exchange that fails, or hangs past
    # --pbt-timeout seconds (e.g. a collective on a broken multi-GPU fabric), is reported in the
    # line's pbt_exchange instead of costing the measured throughput line
    pbt = None
    if pop >= 4:
        def on_timeout():
            if rank == 0 and line is not None:
                line["pbt_exchange"] = {"error": f"timeout after {args.pbt_timeout} s"}
                print(json.dumps(line), flush=True)
            os._exit(0)
        watchdog = threading.Timer(args.pbt_timeout, on_timeout)
        watchdog.daemon = True
        watchdog.start()
        try:
            from paper_2206_08888_b200.dist import Comm, NativeShardedPBT
            comm = (Comm.nccl(device=gpu) if (world > 1 and backend == "nccl")
                    else Comm.host(device=gpu) if world > 1 else None)
            if comm is None:  # single rank: a one-rank host transport (no communication)
                comm = _solo_comm(gpu)
            pstate = pb.PBTState(n)
            rng = pb.RngSequence(SEED, 0, "kDonorChoice")
            ex = NativeShardedPBT(st, hy, comm)
            times, parts, plans = [], [], []
            for ev in range(3):
                for m in range(n):
                    g = off + m
                    pstate.record_return(m, pb.RngStream.of(SEED, g, "kGeneric", ev).uniform(0))
                st.synchronize()
                barrier()
                t0 = time.perf_counter()
                plan = ex.evolve(pstate, rng)
                dt = (time.perf_counter() - t0) * 1e3
                times.append(max_over_ranks(dt))
                parts.append(ex.last_exchange_ms)
                plans.append(plan)
            per = pop // world if args.scaling == "strong" else n
            cross = [sum(1 for d, s_ in zip(p.replaced, p.donors) if d // per != s_ // per)
                     for p in plans]
            blob = pb.pbrl.member_blob_size(st) * 4
            med = sorted(times)[1]
            pbt = {"ms": med, "samples_ms": times, "transport": comm.kind,
                   "breakdown_ms_rank0": parts[1], "replaced": len(plans[1].replaced),
                   "cross_rank_copies": cross[1], "blob_bytes": blob,
                   "interval_updates": args.pbt_interval,
                   "amortised_share_of_step_time": med / (args.pbt_interval * total_ms / K)}
            comm.close()
        except Exception as e:  # reported, not fatal: the throughput line stands on its own
            pbt = {"error": f"{type(e).__name__}: {e}"}
        finally:
            watchdog.cancel()
    if line is not None:
        line["pbt_exchange"] = pbt
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def _solo_comm(gpu):
    """A one-rank host transport: the all-gather is a copy, there is nothing to exchange."""
    import ctypes as C_
    import numpy as np
    from paper_2206_08888_b200 import _lib
    from paper_2206_08888_b200.dist import Comm

    def allgather(_ctx, send, count, recv):
        np.ctypeslib.as_array(recv, (count,))[:] = np.ctypeslib.as_array(send, (count,))
        return 0

    def exchange(_ctx, ops, n_ops):
        return 0 if n_ops == 0 else 1

    ag, ex = _lib.ALLGATHER_FN(allgather), _lib.EXCHANGE_FN(exchange)
    ops = _lib.CommOps(None, ag, ex)
    h = C_.c_void_p()
    _lib.call("pbrl_comm_create_host", C_.byref(ops), 0, 1, gpu, C_.byref(h))
    return Comm(h, 0, 1, "host (single rank)", keep=(ag, ex, ops))


if __name__ == "__main__":
    main()
