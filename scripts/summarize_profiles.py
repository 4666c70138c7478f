#!/usr/bin/env python3
"""Turn the scratch outputs of scripts/gpu_round_artifacts.sh (gpurun_out/) into
the committed summaries under profiles/:

  launches.csv        -> <prefix>_launches_config4_summary.json (per-kernel share of GPU time)
  guard_full.ncu-rep  -> <prefix>_guard_kernel_ncu.json
  tc_full.ncu-rep     -> <prefix>_tc_kernel_ncu.json (when the capture finished)
  bench.json / bench_ref.json / configs.jsonl -> copied

usage: python scripts/summarize_profiles.py [--prefix r2] [--src gpurun_out]
"""
import argparse
import csv
import json
import shutil
import subprocess
from collections import defaultdict
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
METRICS = [
    "gpu__time_duration.sum", "sm__cycles_elapsed.avg", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_elapsed",
    "smsp__warp_issue_stalled_long_scoreboard_per_warp_active.pct",
    "smsp__warp_issue_stalled_barrier_per_warp_active.pct",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__m_xbar2l1tex_read_bytes.sum",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "launch__shared_mem_per_block_dynamic", "launch__cluster_dim_x", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def launch_summary(path: Path, command: str) -> dict:
    tot = defaultdict(float)
    cnt = defaultdict(int)
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    for row in csv.DictReader(lines):
        if row["Metric Name"] != "gpu__time_duration.sum":
            continue
        name = row["Kernel Name"].split("(")[0].replace("void ", "")
        tot[name] += float(row["Metric Value"].replace(",", ""))
        cnt[name] += 1
    all_t = sum(tot.values())
    ks = sorted(tot, key=lambda k: -tot[k])
    return {"unit": "ns", "command": command,
            "note": "serialised, cold-cache per-launch times; 5 frames (3 warm-up + 2 timed) plus torch fills (L2 flush)",
            "kernels": [{"kernel": k, "launches": cnt[k], "total": tot[k], "avg": tot[k] / cnt[k],
                         "share": round(tot[k] / all_t, 4)} for k in ks]}


def rep_summary(rep: Path, kernel: str, capture: str, launch: str) -> dict:
    out = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units, vals = rows[0], rows[1], rows[2]
    m = {}
    for name in METRICS:
        if name in hdr:
            i = hdr.index(name)
            m[name] = {"value": vals[i], "unit": units[i]}
    def nbytes(k):
        v = m.get(k)
        return float(v["value"].replace(",", "")) * SCALE.get(v["unit"], 1) if v else 0.0
    return {"kernel": kernel, "capture": capture, "launch": launch,
            "dram_bytes_per_launch": nbytes("dram__bytes_read.sum") + nbytes("dram__bytes_write.sum"), "metrics": m}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--prefix", default="r2")
    ap.add_argument("--src", default=str(ROOT / "gpurun_out"))
    a = ap.parse_args()
    src, dst = Path(a.src), ROOT / "profiles"
    p = a.prefix
    if (src / "launches.csv").exists():
        s = launch_summary(src / "launches.csv", "ncu --metrics gpu__time_duration.sum --clock-control none -c 400 "
                           "python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e")
        (dst / f"{p}_launches_config4_summary.json").write_text(json.dumps(s, indent=1) + "\n")
        shutil.copy(src / "launches.csv", dst / f"{p}_launches_config4.csv")
    base = "python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
    if (src / "train_launches.csv").exists():
        s = launch_summary(src / "train_launches.csv", "ncu --metrics gpu__time_duration.sum --clock-control none "
                           "-c 2000 python scripts/train_profile.py 3")
        s["note"] = "serialised, cold-cache per-launch times; 3 paper-profile training iterations (batch 4096)"
        (dst / f"{p}_launches_train_summary.json").write_text(json.dumps(s, indent=1) + "\n")
    for rep, kern, cap, out in [
            ("guard_tc_kernel_full.ncu-rep", "guard_tc_kernel", "--set full -k regex:guard_tc_kernel", "guard"),
            ("resolve_shade_kernel_full.ncu-rep", "resolve_shade_kernel", "--set full -k regex:resolve_shade_kernel",
             "resolve_shade"),
            ("setup_kernel_full.ncu-rep", "setup_kernel", "--set full -k regex:setup_kernel", "setup"),
            ("gemm_full.ncu-rep", "gemm_tf32x3_kernel (trainer, forward body layer 4096 x 256 x 256)",
             "--set full -k regex:gemm_tf32x3 -s 105 -c 1 python scripts/train_profile.py 2", "train_gemm"),
            ("tc_full.ncu-rep", "nedf_mlp_tc_kernel (cluster-multicast pair, as benchmarked)",
             "--metrics <list in scripts/gpu_round_artifacts.sh> -k regex:nedf_mlp_tc_kernel", "tc"),
            ("tc_single_full.ncu-rep", "nedf_mlp_tc_kernel (single-CTA variant)",
             "--set full -k regex:nedf_mlp_tc_kernel [--tc-kernel single]", "tc_single_full"),
            ]:
        if (src / rep).exists() and (src / rep).stat().st_size > 0:
            if out != "tc":      # full-set captures: also the section details (rules, speed-of-light, stalls)
                det = subprocess.run(["ncu", "-i", str(src / rep), "--page", "details", "--csv"], capture_output=True,
                                     text=True).stdout
                if det:
                    name = "tc_single" if out == "tc_single_full" else out
                    (dst / f"{p}_{name}_kernel_details.csv").write_text(det)
            try:
                s = rep_summary(src / rep, kern, f"ncu {cap} --clock-control none" +
                                ("" if "train_profile" in cap else f" -s 2 -c 1 {base}"),
                                "trainer GEMM" if out == "train_gemm" else "STEP-1 launch of a config-4 frame")
                (dst / f"{p}_{out}_kernel_ncu.json").write_text(json.dumps(s, indent=1) + "\n")
            except (subprocess.CalledProcessError, IndexError) as e:
                print("skip", rep, e)
    for f, t in [("bench.json", f"{p}_bench_config4.json"), ("bench_ref.json", f"{p}_bench_reference_arm.json"),
                 ("configs.jsonl", f"{p}_configs.jsonl")]:
        if (src / f).exists():
            lines = [l for l in (src / f).read_text().splitlines() if l.startswith("{")]
            if lines:
                (dst / t).write_text(("\n".join(lines) if f.endswith("l") else lines[-1]) + "\n")
    print("profiles updated:", sorted(x.name for x in dst.iterdir()))


if __name__ == "__main__":
    main()
