"""Summarise an `ncu --set full` report: one CSV row per kernel launch with the
metrics the round README quotes, and (optionally) the traffic JSON bench.py
reads for roofline.traffic.

    python scripts/ncu_summary.py REPORT.ncu-rep OUT.csv [TRAFFIC.json BATCH WORKLOAD]
"""
import csv
import io
import json
import subprocess
import sys

METRICS = {
    "gpu__time_duration.sum": "time_ns",
    "dram__bytes_read.sum": "dram_read_B",
    "dram__bytes_write.sum": "dram_write_B",
    "FBSP.TriageCompute.dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
    "sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active": "tensor_pct",
    "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_active": "tmem_tensor_pct",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active": "xu_pct",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active": "fma_pct",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active": "alu_pct",
    "sm__issue_active.avg.pct_of_peak_sustained_elapsed": "issue_pct",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed": "smem_pct",
    "sm__cycles_elapsed.avg.per_second": "sm_hz",
}
CLASS = [("attn_tc", "tile_attention"), ("mlp_tc", "mlp_fused"), ("block_tc", "block_tail"), ("layernorm", "layernorm"),
         ("stitch", "stitch_residual"), ("gather", "tile_gather")]


def kernel_class(name, ln):
    for key, cls in CLASS:
        if key in name:
            return cls
    if "gemm_tc_kernel" in name:
        return f"gemm<{name.split('gemm_tc_kernel<')[1].split('>')[0]}>" if "<" in name else "gemm"
    return name[:40]


def main():
    rep, out = sys.argv[1], sys.argv[2]
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    ik = hdr.index("Kernel Name")
    scale = {"ns": 1.0, "us": 1e3, "ms": 1e6, "nsecond": 1.0, "usecond": 1e3, "msecond": 1e6, "second": 1e9,
             "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    recs = []
    for r in data:
        rec = {"kernel": kernel_class(r[ik], None), "name": r[ik][:120]}
        for m, short in METRICS.items():
            if m not in hdr:
                rec[short] = ""
                continue
            v, u = r[hdr.index(m)], units[hdr.index(m)]
            if u in scale and v not in ("", "n/a"):   # normalise to ns / bytes
                v = repr(float(v.replace(",", "")) * scale[u])
            rec[short] = v
        recs.append(rec)
    with open(out, "w", newline="") as f:
        w = csv.DictWriter(f, fieldnames=list(recs[0].keys()))
        w.writeheader()
        w.writerows(recs)
    for rec in recs:
        print(f"{rec['kernel']:24s} {float(rec['time_ns'] or 0) / 1e3:8.1f} us  "
              f"tensor {float(rec['tmem_tensor_pct'] or 0):5.1f}%  xu {float(rec['xu_pct'] or 0):5.1f}%  "
              f"fma {float(rec['fma_pct'] or 0):5.1f}%  issue {float(rec['issue_pct'] or 0):5.1f}%  "
              f"dram {(float(rec['dram_read_B'] or 0) + float(rec['dram_write_B'] or 0)) / 1e6:8.1f} MB "
              f"= {(float(rec['dram_read_B'] or 0) + float(rec['dram_write_B'] or 0)) / max(float(rec['time_ns'] or 1), 1):6.0f} GB/s")
    if len(sys.argv) > 5:
        tj, batch, wl = sys.argv[3], int(sys.argv[4]), sys.argv[5]
        traffic = {}
        for rec in recs:
            if rec["kernel"] == "tile_attention" and rec["dram_read_B"]:
                traffic["tile_attention"] = {
                    "dram_bytes_per_launch": float(rec["dram_read_B"]) + float(rec["dram_write_B"]),
                    "batch": batch, "workload": wl}
                break
        json.dump(traffic, open(tj, "w"), indent=1)
        print("wrote", tj, traffic)


if __name__ == "__main__":
    main()
