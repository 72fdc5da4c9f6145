"""Summarise one ncu --set full capture of a bank step into profiles/:

  python tools/profile_summary.py gpurun_out/prof_r01.ncu-rep profiles/r01

writes <prefix>_kernels.json (per kernel + per bench phase: duration, DRAM
bytes, tensor-pipe / SM / memory throughput) and <prefix>_ncu_summary.txt.
"""
import csv
import io
import json
import subprocess
import sys

METRICS = {
    "duration_us": "gpu__time_duration.sum",
    "dram_read": "dram__bytes_read.sum",
    "dram_write": "dram__bytes_write.sum",
    "dram_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "tensor_pct": "sm__ops_path_tensor_op_utchmma_src_tf32_dst_fp32_sparsity_off.sum.pct_of_peak_sustained_elapsed",
    "smem_lsu_pct": "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "l2_pct": "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm_pct": "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "mem_pct": "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
    "regs": "launch__registers_per_thread",
    "grid": "launch__grid_size",
    "block": "launch__block_size",
}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1.0,
         "usecond": 1.0, "ms": 1e3, "msecond": 1e3}


SIDE = ("mmd_prep", "beta_finish", "bias_from_partials", "head_dw", "ce_loss")  # side-stream launches


def phase_of(name, in_mmd=False):
    if any(s in name for s in SIDE):
        return "side_stream"  # overlapped with the main stream in the bench (serialised under ncu)
    if in_mmd or "mmd_w_kernel" in name or "mmd_wsum" in name:
        return "mmd_pairs"  # the materialised-W path: pass 1, Wsum, V = W.Z GEMM
    if "umma_kernel<0, 1" in name or "head_fwd" in name:
        return "fwd_gemm"
    if "umma_kernel<0, 0" in name or "gemm_simt" in name or "head_dx" in name:
        return "dx_gemm"
    if "umma_kernel<1, 1" in name or "head_dw" in name:
        return "dw_gemm"
    if "mmd_tc" in name:
        return "mmd_pairs"
    if "beta_" in name or "mmd_prep" in name:
        return "mmd_beta"
    if "ce_kernel" in name or "row_sum" in name or "ce_loss" in name:
        return "ce"
    if "bias_sgd" in name or "bias_from_partials" in name:
        return "bias_sgd"
    return "other"


def main(rep, prefix):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    col = {h: i for i, h in enumerate(hdr)}
    kernels = []
    in_mmd = False
    for r in rows[2:]:
        k = {"name": r[col["Kernel Name"]]}
        for key, metric in METRICS.items():
            i = col.get(metric, next((j for h, j in col.items() if h.endswith(metric)), None))
            if i is None or not r[i]:
                continue
            try:
                v = float(r[i].replace(",", ""))
            except ValueError:
                continue
            u = units[i]
            if key.startswith("dram_") and key != "dram_pct":
                v *= SCALE.get(u, 1)
            if key == "duration_us":
                v *= SCALE.get(u, 1)
            k[key] = v
        if "mmd_w_kernel" in k["name"]:
            in_mmd = True
        if "mmd_finish" in k["name"]:
            in_mmd = False
        k["phase"] = phase_of(k["name"], in_mmd)
        kernels.append(k)
    phases = {}
    for k in kernels:
        p = phases.setdefault(k["phase"], {"kernels": 0, "duration_us": 0.0,
                                           "dram_bytes_per_step": 0.0})
        p["kernels"] += 1
        p["duration_us"] += k.get("duration_us", 0.0)
        p["dram_bytes_per_step"] += k.get("dram_read", 0.0) + k.get("dram_write", 0.0)
    out = {"capture": rep, "note": "one bank step (C2, G=32) under ncu --set full "
                                   "--clock-control none: cold-cache, serialised; compare shares",
           "kernels": kernels, "phases": phases}
    with open(prefix + "_kernels.json", "w") as f:
        json.dump(out, f, indent=1)
    tot = sum(k.get("duration_us", 0) for k in kernels)
    lines = [f"ncu --set full capture: {rep}", "one bank step, C2 x 32 models, per kernel (tf32% = tf32 tensor-op rate vs peak):",
             f"{'us':>9} {'share':>6} {'DRAM MB':>9} {'dram%':>6} {'tf32%':>6} {'L2%':>5} {'SM%':>6}  kernel"]
    for k in kernels:
        lines.append(f"{k.get('duration_us', 0):9.1f} {100 * k.get('duration_us', 0) / tot:5.1f}% "
                     f"{(k.get('dram_read', 0) + k.get('dram_write', 0)) / 1e6:9.1f} "
                     f"{k.get('dram_pct', 0):6.1f} {k.get('tensor_pct', 0):6.1f} {k.get('l2_pct', 0):5.1f} "
                     f"{k.get('sm_pct', 0):6.1f}  {k['name'][:90]}")
    lines.append(f"{tot:9.1f}  total")
    lines.append("per phase: " + json.dumps({p: {"us": round(v["duration_us"], 1),
                                                 "dram_MB": round(v["dram_bytes_per_step"] / 1e6, 1)}
                                             for p, v in phases.items()}))
    with open(prefix + "_ncu_summary.txt", "w") as f:
        f.write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
