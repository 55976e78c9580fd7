"""FP64 roofline evidence from ncu for the K4 pipeline kernels (SURVEY.md
§8(d): FP64 instruction counts, FP64-pipe utilisation, divergence, DRAM).

  python tools/ncu_fp64.py parse <ncu long-format csv> <pairs> <out.json> [workload note]

The csv comes from
  ncu --metrics <METRICS> --clock-control none --csv --log-file X.csv \
      python tools/prof_target.py <workload> ...
Per kernel (summed over launches): time, DFMA/DADD/DMUL thread instructions
(predicated on), FP64-pipe active % (time-weighted), threads per instruction,
DRAM bytes. Totals over the K4 kernels (k_pre_class, k_sig_*, k_pipe_*):
flops = 2 DFMA + DADD + DMUL, flops per pair, the time-weighted FP64-pipe
fraction, DRAM bytes per pair. ncu times are serialised, cold-cache and
taken under replay: only the shares and the counts are used, never a rate.
"""
import csv
import json
import sys
from collections import defaultdict

METRICS = ["gpu__time_duration.sum",
           "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum",
           "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum",
           "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum",
           "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
           "smsp__thread_inst_executed_per_inst_executed.ratio",
           "sm__warps_active.avg.pct_of_peak_sustained_active",
           "dram__bytes_read.sum", "dram__bytes_write.sum"]
K4 = ("k_pre_class", "k_sig_", "k_pipe_", "k_edge_pairs")


def num(s):
    return float(s.replace(",", "")) if s not in ("", "n/a") else 0.0


def scale(unit):
    return {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-6, "usecond": 1e-3,
            "msecond": 1.0, "second": 1e3, "ns": 1e-6, "us": 1e-3, "ms": 1.0}.get(unit, 1.0)


def parse(path, pairs, out, note=""):
    rows = list(csv.reader(open(path)))
    start = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    hdr = rows[start]
    iI, iN, iM, iU, iV = (hdr.index(c) for c in ("ID", "Kernel Name", "Metric Name", "Metric Unit", "Metric Value"))
    launch = defaultdict(dict)
    names = {}
    for r in rows[start + 1:]:
        if len(r) <= iV:
            continue
        launch[r[iI]][r[iM]] = num(r[iV]) * scale(r[iU])
        names[r[iI]] = r[iN].split("(")[0].replace("void ", "").strip()
    per = defaultdict(lambda: defaultdict(float))
    for lid, m in launch.items():
        n = names[lid]
        t = m.get("gpu__time_duration.sum", 0.0)  # ms
        p = per[n]
        p["launches"] += 1
        p["ms"] += t
        for key in ("dfma", "dadd", "dmul"):
            p[key] += m.get(f"smsp__sass_thread_inst_executed_op_{key}_pred_on.sum", 0.0)
        p["fp64_pct_x_ms"] += m.get("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", 0.0) * t
        p["tpi_x_ms"] += m.get("smsp__thread_inst_executed_per_inst_executed.ratio", 0.0) * t
        p["occ_x_ms"] += m.get("sm__warps_active.avg.pct_of_peak_sustained_active", 0.0) * t
        p["dram"] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
    kernels = {}
    tot = defaultdict(float)
    for n, p in sorted(per.items(), key=lambda x: -x[1]["ms"]):
        flops = 2 * p["dfma"] + p["dadd"] + p["dmul"]
        k = {"launches": int(p["launches"]), "ms": p["ms"], "flops": flops, "dfma": p["dfma"], "dadd": p["dadd"],
             "dmul": p["dmul"], "fp64_pipe_pct": p["fp64_pct_x_ms"] / p["ms"] if p["ms"] else 0.0,
             "threads_per_inst": p["tpi_x_ms"] / p["ms"] if p["ms"] else 0.0,
             "warps_active_pct": p["occ_x_ms"] / p["ms"] if p["ms"] else 0.0, "dram_bytes": p["dram"]}
        kernels[n] = k
        if n.startswith(K4):
            tot["ms"] += p["ms"]
            tot["flops"] += flops
            tot["fp64_x_ms"] += p["fp64_pct_x_ms"]
            tot["dram"] += p["dram"]
            for key in ("dfma", "dadd", "dmul"):
                tot[key] += p[key]
    res = {"pairs": pairs, "note": note, "source_csv": path,
           "flops_per_pair": tot["flops"] / pairs, "dfma_per_pair": tot["dfma"] / pairs,
           "dadd_per_pair": tot["dadd"] / pairs, "dmul_per_pair": tot["dmul"] / pairs,
           "fp64_pipe_frac_time_weighted": tot["fp64_x_ms"] / tot["ms"] / 100.0 if tot["ms"] else None,
           "k4_ms_ncu": tot["ms"], "dram_bytes_per_pair": tot["dram"] / pairs,
           "ncu_fp64_tflops_serialised": tot["flops"] / (tot["ms"] * 1e-3) / 1e12 if tot["ms"] else None,
           "kernels": kernels}
    with open(out, "w") as f:
        json.dump(res, f, indent=1)
    print(f"flops/pair {res['flops_per_pair']:.0f}, fp64 pipe (time-weighted) "
          f"{res['fp64_pipe_frac_time_weighted']:.3f}, DRAM B/pair {res['dram_bytes_per_pair']:.0f}")
    for n, k in list(kernels.items())[:14]:
        print(f"  {n:40s} {k['launches']:4d} {k['ms']:9.3f} ms  fp64 {k['fp64_pipe_pct']:5.1f}%  "
              f"thr/inst {k['threads_per_inst']:5.2f}  flops {k['flops']:.3g}")


if __name__ == "__main__":
    if sys.argv[1] == "metrics":
        print(",".join(METRICS))
    else:
        parse(sys.argv[2], int(sys.argv[3]), sys.argv[4], sys.argv[5] if len(sys.argv) > 5 else "")
