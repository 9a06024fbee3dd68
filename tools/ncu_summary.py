"""Summarise an `ncu --set full` capture of one CaffeNet training step's tensor-core launches.

    ncu -i prof_step_gemm.ncu-rep --page raw --csv > raw.csv
    python tools/ncu_summary.py raw.csv [--launches launches_step.csv] [--out profiles/rNN_ncu_summary.json]

Labels the 23 GEMM launches in the order tools/one_step.py issues them (forward conv1-5, fc6-8;
backward fc8..fc6 weight/data gradient, conv5..conv2 weight/data gradient, conv1 weight gradient)
and extracts time, algorithmic TFLOP/s (SURVEY App. A FLOPs), tensor-pipe activity, L2->SM bytes,
DRAM bytes, shared-memory store wavefronts, global store efficiency and the SM clock.
"""
import argparse
import csv
import json

# algorithmic GFLOP per pass at batch 256 (2 * MACs)
CONV_GF = {"conv1": 53.97, "conv2": 114.66, "conv3": 76.55, "conv4": 57.42, "conv5": 38.28}
FC_GF = {"fc6": 2 * 256 * 9216 * 4096 / 1e9, "fc7": 2 * 256 * 4096 * 4096 / 1e9, "fc8": 2 * 256 * 4096 * 1000 / 1e9}
# backward launch order per layer: data gradient first (nets.Net.dgrad_first, the default since
# round 2's end; --wgrad-first for captures of the earlier schedule)
_P = ("wgrad", "dgrad") if "--wgrad-first" in __import__("sys").argv else ("dgrad", "wgrad")
ORDER = ([f"conv{i} fwd" for i in range(1, 6)] + ["fc6 fwd", "fc7 fwd", "fc8 fwd"] +
         [f"{l} {p}" for l in ("fc8", "fc7", "fc6") for p in _P] +
         [f"conv{i} {p}" for i in (5, 4, 3, 2) for p in _P] + ["conv1 wgrad"])

COLS = {
    "time_us": ("gpu__time_duration.sum", 1e-3),
    "tensor_pipe_active_pct": ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", 1),
    "bf16_tensor_op_pct": ("sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32_sparsity_off.avg.pct_of_peak_sustained_elapsed", 1),
    "l2_to_sm_MB": ("l1tex__m_xbar2l1tex_read_bytes.sum", 1e-6),
    "dram_read_MB": ("dram__bytes_read.sum", 1e-6),
    "dram_write_MB": ("dram__bytes_write.sum", 1e-6),
    "smem_st_wavefronts": ("l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum", 1),
    "gst_requests": ("l1tex__t_requests_pipe_lsu_mem_global_op_st.sum", 1),
    "gst_sectors": ("l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum", 1),
    "gst_wavefronts_pct": ("l1tex__t_output_wavefronts_pipe_lsu_mem_global_op_st.sum.pct_of_peak_sustained_elapsed", 1),
    "sm_clock_GHz": ("sm__cycles_elapsed.avg.per_second", 1e-9),
    "grid": ("launch__grid_size", 1),
}


def num(s):
    try:
        return float(s.replace(",", ""))
    except ValueError:
        return None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("raw")
    ap.add_argument("--launches", default=None)
    ap.add_argument("--out", default=None)
    ap.add_argument("--wgrad-first", action="store_true", help="capture of the weight-gradient-first schedule")
    args = ap.parse_args()
    rows = list(csv.reader(open(args.raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    idx = {h: i for i, h in enumerate(hdr)}
    out = []
    for k, r in enumerate(data):
        label = ORDER[k] if len(data) == len(ORDER) else f"launch {k}"
        rec = {"launch": label, "kernel": r[idx["Kernel Name"]].split("(")[0]}
        for key, (col, scale) in COLS.items():
            if col in idx:
                v = num(r[idx[col]])
                # ncu reports time in the unit of row 2 (ns / us / ms)
                if key == "time_us" and v is not None:
                    u = units[idx[col]]
                    v = v * {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "msecond": 1e3, "nsecond": 1e-3}.get(u, 1e-3)
                elif v is not None:
                    u = units[idx[col]].lower()
                    if u.endswith("byte"):      # report MB
                        v = v * {"byte": 1e-6, "kbyte": 1e-3, "mbyte": 1.0, "gbyte": 1e3}.get(u, 1.0)
                    elif u.endswith("hz"):      # report GHz
                        v = v * {"hz": 1e-9, "khz": 1e-6, "mhz": 1e-3, "ghz": 1.0}.get(u, 1.0)
                    else:
                        v = v * scale
                rec[key] = round(v, 3) if v is not None else None
        lay, p = label.split(" ")[0], label.split(" ")[-1]
        gf = CONV_GF.get(lay, FC_GF.get(lay))
        if gf and rec.get("time_us"):
            rec["algorithmic_tflops"] = round(gf * 1e9 / (rec["time_us"] * 1e-6) / 1e12, 1)
        if rec.get("l2_to_sm_MB") and rec.get("time_us"):
            rec["l2_to_sm_TBps"] = round(rec["l2_to_sm_MB"] * 1e6 / (rec["time_us"] * 1e-6) / 1e12, 2)
        out.append(rec)
    res = {"captured": "ncu --set full --import-source on --clock-control none --profile-from-start off "
                       "-k 'regex:tc_gemm|tc_halo' python tools/one_step.py (tools/_ncu_round.sh)",
           "note": "ncu replays each kernel; times are cold-cache per launch (compare shares, not absolutes)",
           "gemm_launches": out}
    if args.launches:
        lines = [l for l in open(args.launches) if not l.startswith("==")]
        lrows = list(csv.reader(lines))
        h = lrows[0]
        ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
        ui = h.index("Metric Unit")
        by = {}
        tot = 0.0
        n = 0
        for r in lrows[1:]:
            if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
                continue
            v = num(r[vi]) * {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(r[ui], 1e-3)
            name = r[ki].split("(")[0].replace("void ", "").replace("cb::", "")
            by[name] = by.get(name, 0.0) + v
            tot += v
            n += 1
        res["launch_list_summary"] = {"launches": n, "total_us": round(tot, 1),
                                      "by_kernel_us": {k: round(v, 1) for k, v in sorted(by.items(), key=lambda x: -x[1])}}
    # conv GEMM aggregates for bench.py's roofline: mean DRAM bytes per launch and the tensor-pipe
    # activity weighted by each launch's algorithmic FLOPs
    conv = [r for r in out if r["launch"].startswith("conv")]
    if conv and all(r.get("dram_read_MB") is not None for r in conv):
        fl = [CONV_GF[r["launch"].split(" ")[0]] for r in conv]
        tp = [r.get("tensor_pipe_active_pct") or 0.0 for r in conv]
        res["conv_gemm_aggregate"] = {
            "conv_gemm_launches": len(conv),
            "conv_gemm_dram_bytes_per_launch": sum((r["dram_read_MB"] + r["dram_write_MB"]) * 1e6 for r in conv) / len(conv),
            "conv_gemm_tensor_pipe_pct_flop_weighted": sum(f * t for f, t in zip(fl, tp)) / sum(fl),
            "conv_gemm_tensor_pipe_pct_time_weighted": sum((r.get("time_us") or 0) * t for r, t in zip(conv, tp)) /
            max(1e-9, sum(r.get("time_us") or 0 for r in conv)),
        }
    s = json.dumps(res, indent=1)
    if args.out:
        open(args.out, "w").write(s + "\n")
    for rec in out:
        print(f"{rec['launch']:14s} {rec.get('time_us', 0):8.1f} us  {rec.get('algorithmic_tflops', 0):7.1f} TF  "
              f"tc {rec.get('tensor_pipe_active_pct') or 0:5.1f}%  bf16op {rec.get('bf16_tensor_op_pct') or 0:5.1f}%  "
              f"L2->SM {rec.get('l2_to_sm_TBps') or 0:5.2f} TB/s  dram r/w {rec.get('dram_read_MB') or 0:6.1f}/"
              f"{rec.get('dram_write_MB') or 0:6.1f} MB  smem_st {rec.get('smem_st_wavefronts') or 0:9.0f}  "
              f"gst req/sec {rec.get('gst_requests') or 0:8.0f}/{rec.get('gst_sectors') or 0:9.0f}  "
              f"clk {rec.get('sm_clock_GHz') or 0:4.2f}")
    if "launch_list_summary" in res:
        print(json.dumps(res["launch_list_summary"])[:1500])


if __name__ == "__main__":
    main()
