#!/usr/bin/env python3
"""Summarise the ncu captures of tools/profile_round.sh (gpurun_out/prof/) into profiles/:
per-kernel duration, DRAM bytes, pipe utilisation, achieved vs algorithmic bytes / flops, and the
launch list of the bench command.  Run here (no GPU needed): python tools/summarize_profiles.py r01
"""
from __future__ import annotations

import csv
import io
import json
import shutil
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
SRC = ROOT / "gpurun_out" / "prof"
DST = ROOT / "profiles"

METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
    "SM_C.TriageCompute.smsp__pipe_tensor_subpipe_dmma_cycles_active.avg", "sm__cycles_elapsed.avg",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
    "sm__ops_path_tensor_op_utchmma_src_tf32_dst_fp32_sparsity_off.sum.pct_of_peak_sustained_elapsed",
    "sm__ops_path_tensor_op_utchmma_src_fp16_dst_fp32_sparsity_off.sum.pct_of_peak_sustained_elapsed",
    "sm__ops_path_tensor_op_utchmma_src_fp16_dst_fp32_sparsity_off.sum.pct_of_peak_sustained_active",
    "sm__ops_path_tensor_op_utchmma_src_tf32_dst_fp32_sparsity_off.sum.pct_of_peak_sustained_active",
    "sm__pipe_tensor_op_utchmma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active",
]


def raw(rep: Path):
    out = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    kernels = []
    for vals in rows[2:]:
        d = {"kernel": vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"}
        for h, u, v in zip(hdr, units, vals):
            if h in METRICS:
                try:
                    d[h] = float(v.replace(",", ""))
                except ValueError:
                    d[h] = v
                d[h + ".unit"] = u
        kernels.append(d)
    return kernels


def to_bytes(v, unit):
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
    return v * scale


def to_us(v, unit):
    return v * {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "nsecond": 1e-3, "ms": 1e3, "msecond": 1e3}.get(unit, 1.0)


def main():
    tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
    DST.mkdir(exist_ok=True)
    summary = {"round": tag, "source": "tools/profile_round.sh on 1 B200 (gpurun), ncu --set full --clock-control none",
               "kernels": {}}
    traffic = {}
    for name, rep in (("eval_f64_multi", "eval_multi.ncu-rep"), ("eval_f64_dmma", "eval_f64.ncu-rep"),
                      ("eval_f32_umma_sk", "eval_f32.ncu-rep"),
                      ("de_runs", "runs.ncu-rep"), ("updates", "updates.ncu-rep"),
                      ("updates", "pso_update.ncu-rep"), ("de_run", "de_run.ncu-rep")):
        p = SRC / rep
        if not p.exists():
            continue
        for k in raw(p):
            kn = k["kernel"]
            dur = to_us(k.get("gpu__time_duration.sum", 0.0), k.get("gpu__time_duration.sum.unit", "ns"))
            rd = to_bytes(k.get("dram__bytes_read.sum", 0.0), k.get("dram__bytes_read.sum.unit", "byte"))
            wr = to_bytes(k.get("dram__bytes_write.sum", 0.0), k.get("dram__bytes_write.sum.unit", "byte"))
            e = {"duration_us": dur, "dram_read_bytes": rd, "dram_write_bytes": wr,
                 "dram_GBps": (rd + wr) / (dur * 1e-6) / 1e9 if dur else None}
            for m in METRICS[3:]:
                if m in k:
                    e[m] = k[m]
            if name == "eval_f64_dmma":
                e["algorithmic_flop"] = 2.0 * 1000 * 1000 * 1024
                e["achieved_TFLOPs_under_ncu"] = e["algorithmic_flop"] / (dur * 1e-6) / 1e12
                traffic["eval_f64_dmma_kernel"] = rd + wr
            if name == "eval_f64_multi":
                e["algorithmic_flop"] = 3 * 2.0 * 1000 * 1000 * 1024
                e["achieved_TFLOPs_under_ncu"] = e["algorithmic_flop"] / (dur * 1e-6) / 1e12
                traffic["eval_f64_dmma_multi_kernel"] = rd + wr
            if name == "eval_f32_umma_sk":
                e["algorithmic_flop"] = 2.0 * 1000 * 1000 * 1024
                e["achieved_TFLOPs_under_ncu"] = e["algorithmic_flop"] / (dur * 1e-6) / 1e12
                traffic["eval_f32_umma_sk_kernel"] = rd + wr
            if "pso_update" in kn:
                traffic["pso_update_vec_kernel"] = rd + wr
                e["algorithmic_bytes"] = 5 * 8 * 16384 * 1000
                e["algorithmic_GBps"] = e["algorithmic_bytes"] / (dur * 1e-6) / 1e9
            if "de_trial" in kn:
                traffic["de_trial_stage_kernel"] = rd + wr
                e["algorithmic_bytes"] = 5 * 8 * 16384 * 1000
                e["algorithmic_GBps"] = e["algorithmic_bytes"] / (dur * 1e-6) / 1e9
            key = f"{name}:{kn[:90]}"
            i = 2
            while key in summary["kernels"]:
                key = f"{name}:{kn[:90]}#{i}"
                i += 1
            summary["kernels"][key] = e
    (DST / f"ncu_summary_{tag}.json").write_text(json.dumps(summary, indent=1))
    old = json.loads((DST / "traffic.json").read_text()) if (DST / "traffic.json").exists() else {}
    old.update(traffic)
    (DST / "traffic.json").write_text(json.dumps(old, indent=1))
    lc = SRC / "bench_launches.csv"
    if lc.exists():
        shutil.copy(lc, DST / f"bench_launches_{tag}.csv")
    for name in ("eval_multi", "eval_f64", "eval_f32", "runs", "updates", "pso_update", "de_run"):
        rep = SRC / f"{name}.ncu-rep"
        if rep.exists():
            shutil.copy(rep, DST / f"{name}_{tag}.ncu-rep")
    for f in ("hbm_plain.json", "bench_plain.log", "de_run_plain.log", "runs_plain.log"):
        if (SRC / f).exists():
            shutil.copy(SRC / f, DST / f"{Path(f).stem}_{tag}{Path(f).suffix}")
    print(json.dumps(summary, indent=1)[:6000])


if __name__ == "__main__":
    main()
