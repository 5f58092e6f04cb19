"""Summarise ncu captures for profiles/ (run here, on the CPU, on reports
brought back from the GPU box).

  python tools/ncu_summary.py full  gpurun_out/prof.ncu-rep  > profiles/<name>.json
  python tools/ncu_summary.py list  gpurun_out/launches.csv  > profiles/<name>.json
"""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict

FULL_METRICS = [
    "gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second", "dram__bytes_read.sum",
    "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32_sparsity_off.avg.pct_of_peak_sustained_elapsed",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__m_xbar2l1tex_read_bytes.sum",
    "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic",
    "launch__cluster_dim_x", "smsp__inst_executed.sum",
]


def full(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = []
    for vals in rows[2:]:
        rec = {"kernel": vals[hdr.index("Kernel Name")][:160]}
        for m in FULL_METRICS:
            if m in hdr:
                i = hdr.index(m)
                rec[m] = f"{vals[i]} {units[i]}".strip()
        out.append(rec)
    return out


def launch_list(path):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    i_name, i_val = hdr.index("Kernel Name"), hdr.index("Metric Value")
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows[start + 1:]:
        if len(r) <= i_val:
            continue
        name = r[i_name].split("(")[0][:100]
        agg[name][0] += 1
        agg[name][1] += float(r[i_val].replace(",", ""))
    total = sum(v[1] for v in agg.values()) or 1.0
    return [{"kernel": k, "launches": c, "total_ms": round(t / 1e6, 4), "share": round(t / total, 4)}
            for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1])]


if __name__ == "__main__":
    kind, path = sys.argv[1], sys.argv[2]
    print(json.dumps(full(path) if kind == "full" else launch_list(path), indent=1))
