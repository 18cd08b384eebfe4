"""Phase timeline of the tcgen05 GEMM launches of one TD3 update step (diagnostics).

    PBRL_TC_TRACE=1 python tools/tc_trace.py [--steps S] [--pop N] [--out profiles/x.md]

Runs config-D-shaped TD3 steps (graph-captured, as in bench.py), then reads the per-CTA
globaltimer stamps recorded by k_tc_gemm (TcArgs::trace) for the launches of the last replayed
step and prints, per launch: wall span, setup cost, tiles per CTA, and the median per-tile
phase durations (TMA issue -> first stage landed, MMA, MMA commit -> epilogue start, epilogue).
"""
from __future__ import annotations

import argparse
import ctypes as C
import os
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
EPI = ["store", "bias", "bias_relu", "bias_tanh", "bias_tanh_noise", "relu_mask", "tanh_grad"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=6)
    ap.add_argument("--pop", type=int, default=80)
    ap.add_argument("--out", default=None)
    ap.add_argument("--precision", default="tf32", choices=["tf32", "bf16"])
    ap.add_argument("--dump", type=int, nargs="*", default=[0, 2], help="launches to dump")
    args = ap.parse_args()
    os.environ.setdefault("PBRL_TC_TRACE", "1")
    import torch
    import paper_2206_08888_b200 as pb
    from paper_2206_08888_b200 import _lib

    n, B = args.pop, 256
    st = pb.make_td3_state(n, 17, 6, [256, 256], 1.0, 7, precision=args.precision)
    hy = pb.Td3Hyper.defaults(n)
    st._sync_hyper(hy)
    gb = pb.make_synthetic_batches(4, n, B, 17, 6, 7, device=torch.device("cuda", 0))
    structs = [_lib.Batch(*[x.data_ptr() for x in (b.s, b.a, b.r, b.s2, b.done)]) for b in gb]
    for i in range(args.steps):
        arr = (_lib.Batch * 1)(structs[i % 4])
        _lib.call("pbrl_update_batches_device", st.handle, arr, 1, B, None)
    st.synchronize()

    maxl = 96
    stamps = np.zeros((maxl, 160, 64), dtype=np.uint64)
    meta = np.zeros((maxl, 10), dtype=np.int32)
    cnt = C.c_int()
    _lib.call("pbrl_debug_tc_trace", stamps.ctypes.data_as(C.POINTER(C.c_uint64)),
              meta.ctypes.data_as(C.POINTER(C.c_int)), maxl, C.byref(cnt))
    nl = cnt.value
    lines = [f"# tcgen05 GEMM phase timeline (TD3 pop {n}, 2x256, B={B}, {args.precision}, "
             "last replayed step)", "",
             "| # | tile | op | M,N,K x groups | span us | setup us | tiles/CTA | first TMA->data us"
             " | MMA us | commit->epi us | epilogue us | out-layer wait us | drain us |",
             "|---|---|---|---|---|---|---|---|---|---|---|---|---|"]
    # launches recorded during the first (eager / capture) pass; the captured ones hold the
    # stamps of the last replay
    for li in range(nl):
        s = stamps[li].astype(np.int64)
        used = s[:, 0] > 0
        if not used.any():
            continue
        s = s[used]
        t0 = s[:, 0].min()
        span = (s[:, 63].max() - t0) / 1e3
        setup = np.median(s[:, 1] - s[:, 0]) / 1e3
        ph = {k: [] for k in range(6)}
        tiles = []
        for c in s:
            nt = 0
            for it in range(10):
                b = 2 + 6 * it
                if c[b] == 0 or c[b + 4] == 0:
                    break
                nt += 1
                ph[0].append(c[b + 1] - c[b])
                ph[1].append(c[b + 2] - c[b + 1])
                ph[2].append(c[b + 3] - c[b + 2])
                ph[3].append(c[b + 4] - c[b + 3])
                if c[b + 5]:
                    ph[5].append(c[b + 5] - c[b + 4])
            tiles.append(nt)
            if c[62]:
                last = 2 + 6 * (nt - 1) + 4 if nt else 1
                ph[4].append(c[62] - c[last])
        med = {k: (np.median(v) / 1e3 if v else float("nan")) for k, v in ph.items()}
        m = meta[li]
        op = (f"{EPI[m[8]] if m[8] < len(EPI) else m[8]}" if m[8] != 99 else
              "FWD2 [cols: stage+MMA1 | E1 | MMA2 | E2]") + (f"+out{m[3]}" if m[3] else "")
        lines.append(
            f"| {li} | {m[0]},{'MN' if m[1] else 'K'},{'MN' if m[2] else 'K'} | {op} | "
            f"{m[4]},{m[5]},{m[6]} x {m[7]} | {span:.1f} | {setup:.2f} | "
            f"{min(tiles)}-{max(tiles)} | {med[0]:.2f} | {med[1]:.2f} | {med[2]:.2f} | "
            f"{med[3]:.2f} | {med[5]:.2f} | {med[4]:.2f} |")
    # step timeline: launch windows and the gaps between consecutive GEMM launches
    win = []
    for li in range(nl):
        s = stamps[li].astype(np.int64)
        s = s[s[:, 0] > 0]
        if len(s):
            win.append((li, s[:, 0].min(), s[:, 63].max()))
    win.sort(key=lambda w: w[1])
    lines += ["", "| # | start us | end us | gap before us |", "|---|---|---|---|"]
    t00 = win[0][1] if win else 0
    prev = None
    for li, a, b in win:
        gap = (a - prev) / 1e3 if prev is not None else 0.0
        lines.append(f"| {li} | {(a - t00) / 1e3:.1f} | {(b - t00) / 1e3:.1f} | {gap:.1f} |")
        prev = b
    # per-CTA spread: entry, first tile start (after the PDL wait), exit -- relative to the
    # launch's first CTA entry
    lines += ["", "| # | entry p50/max us | tile0 p50/max us | exit min/p50/max us |",
              "|---|---|---|---|"]
    for li, a, b in win:
        s = stamps[li].astype(np.int64)
        s = s[s[:, 0] > 0]
        e0, t0s, ex = (s[:, 0] - a) / 1e3, (s[:, 2] - a) / 1e3, (s[:, 63] - a) / 1e3
        t0s = t0s[s[:, 2] > 0]
        q = lambda v, f: float(np.percentile(v, f)) if len(v) else float("nan")
        lines.append(f"| {li} | {q(e0, 50):.1f} / {e0.max():.1f} | {q(t0s, 50):.1f} / "
                     f"{q(t0s, 100):.1f} | {ex.min():.1f} / {q(ex, 50):.1f} / {ex.max():.1f} |")
    # raw per-tile stamps (us from the launch's first entry) of the slowest and the median CTA
    for li in args.dump:
        s = stamps[li].astype(np.int64)
        s = s[s[:, 0] > 0]
        if not len(s):
            continue
        a = s[:, 0].min()
        order = np.argsort(s[:, 63])
        lines += ["", f"launch {li}: tile stamps [start, acc1/after waits, E1 done, acc2, E2 done, "
                  "MMA2 issued]"]
        for tag, c in (("slowest", s[order[-1]]), ("median", s[order[len(order) // 2]])):
            tl = []
            for it in range(10):
                b = 2 + 6 * it
                if c[b] == 0:
                    break
                tl.append("[" + ", ".join(f"{(c[b + k] - a) / 1e3:.1f}" if c[b + k] else "-"
                                          for k in range(6)) + "]")
            lines.append(f"  {tag}: entry {(c[0] - a) / 1e3:.1f} " + " ".join(tl) +
                         f" exit {(c[63] - a) / 1e3:.1f}")
    if win:
        busy = sum(b - a for _, a, b in win) / 1e3
        lines.append(f"\nGEMM launches busy {busy:.1f} us of a {(win[-1][2] - t00) / 1e3:.1f} us window")
    txt = "\n".join(lines)
    print(txt)
    if args.out:
        Path(args.out).write_text(txt + "\n")


if __name__ == "__main__":
    main()
