"""Summarise ncu outputs from gpurun_out/ into tracked text under profiles/.

    python profiles/summarize.py <tag> <launches.csv> [<full.ncu-rep> ...]

Writes profiles/<tag>_launches.md (per-step kernel breakdown from the
`--metrics gpu__time_duration.sum` launch list: serialised, cold-cache -- compare shares, not
absolutes), profiles/<tag>_<report>.md (key `--set full` metrics per profiled launch) and
profiles/traffic_<precision>_D.json (DRAM bytes per launch of each kernel class, read by bench.py
as the roofline `traffic` field).
"""
from __future__ import annotations

import collections
import csv
import json
import subprocess
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent

CLASS = [("k_mlp_fwd2", "gemm (tcgen05, fused 2-layer forward)"), ("k_tc_gemm", "gemm (tcgen05)"), ("k_gemm_simt", "gemm (cuda-core)"),
         ("k_out_backward", "output-layer backward"), ("k_fwd_skinny", "output-layer fwd"),
         ("k_dx_skinny", "dX skinny"), ("k_adam", "adam_polyak"), ("k_colsum", "bias grad"),
         ("k_replay_gather", "gather_pack"), ("k_pack_batch", "gather_pack")]


def kclass(name: str) -> str:
    for k, c in CLASS:
        if name.startswith(k) or f" {k}" in name:
            return c
    return "elementwise"


def launches(path: Path, tag: str) -> None:
    rows = list(csv.reader(path.open()))
    hdr, out = None, []
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") == "gpu__time_duration.sum":
                name = d["Kernel Name"].replace("void ", "").split("(")[0]
                out.append((name, d["Grid Size"], float(d["Metric Value"]) / 1e3))
    starts = [i for i, x in enumerate(out) if x[0].startswith("k_td3_step_begin")]
    lines = [f"# {tag}: ncu launch list (gpu__time_duration.sum, --clock-control none)", "",
             "Serialised, cold-cache per-launch times: use the SHARES, not the absolutes.", ""]
    for a, b in zip(starts, starts[1:]):
        seg = out[a:b]
        tot = sum(x[2] for x in seg)
        agg = collections.defaultdict(float)
        for k, g, t in seg:
            agg[kclass(k)] += t
        lines.append(f"## step with {len(seg)} launches: {tot:.1f} us")
        lines.append("")
        lines.append("| class | us | share |")
        lines.append("|---|---|---|")
        for k, t in sorted(agg.items(), key=lambda x: -x[1]):
            lines.append(f"| {k} | {t:.1f} | {100 * t / tot:.1f}% |")
        lines.append("")
        lines.append("| kernel | grid | us |")
        lines.append("|---|---|---|")
        for k, g, t in seg:
            lines.append(f"| `{k}` | {g} | {t:.1f} |")
        lines.append("")
    (HERE / f"{tag}_launches.md").write_text("\n".join(lines))


WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "smsp__inst_executed.sum", "lts__t_sector_hit_rate.pct"]


def full(path: Path, tag: str) -> dict:
    raw = subprocess.run(["ncu", "-i", str(path), "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units = rows[0], rows[1]
    lines = [f"# {tag}: {path.name} (ncu --set full, --clock-control none)", ""]
    traffic = {}
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        name = d.get("Kernel Name", "?").replace("void ", "").split("(")[0]
        lines.append(f"## `{name}` grid {d.get('Grid Size')} block {d.get('Block Size')}")
        for w in WANT:
            if w in d:
                lines.append(f"- {w}: {d[w]} {u.get(w, '')}")
        try:
            rd = float(d["dram__bytes_read.sum"]) * (1e6 if "M" in u["dram__bytes_read.sum"] else
                                                     1e3 if "K" in u["dram__bytes_read.sum"] else
                                                     1e9 if "G" in u["dram__bytes_read.sum"] else 1)
            wr = float(d["dram__bytes_write.sum"]) * (1e6 if "M" in u["dram__bytes_write.sum"] else
                                                      1e3 if "K" in u["dram__bytes_write.sum"] else
                                                      1e9 if "G" in u["dram__bytes_write.sum"] else 1)
            traffic.setdefault(name, []).append(rd + wr)
        except (KeyError, ValueError):
            pass
        lines.append("")
    (HERE / f"{tag}_{path.stem}.md").write_text("\n".join(lines))
    return {k: sum(v) / len(v) for k, v in traffic.items()}


def main():
    tag, csv_path, reps = sys.argv[1], Path(sys.argv[2]), [Path(p) for p in sys.argv[3:]]
    launches(csv_path, tag)
    traffic = {}
    for r in reps:
        traffic.update(full(r, tag))
    prec = "bf16" if "bf16" in tag else ("tf32" if "tf32" in tag else "ffma32")
    cls_map = {"gemm_fwd": ("k_mlp_fwd2", "k_tc_gemm"), "adam_polyak": ("k_adam",)}
    out = {c: next((v for kn in kns for k, v in traffic.items() if k.startswith(kn)), None)
           for c, kns in cls_map.items()}
    out["_note"] = "DRAM bytes per launch (dram__bytes_read.sum + dram__bytes_write.sum) from one ncu --set full capture"
    (HERE / f"traffic_{prec}_D.json").write_text(json.dumps(out, indent=1))
    print("wrote", sorted(p.name for p in HERE.glob(f"{tag}_*")))


if __name__ == "__main__":
    main()
