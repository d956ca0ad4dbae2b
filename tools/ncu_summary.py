"""Summarise an ncu report (--page raw) into the handful of numbers the roofline
needs: duration, DRAM bytes, tensor/DMMA pipe use, occupancy, top stall reasons."""
import csv
import io
import json
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
    "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "launch__occupancy_limit_registers",
    "launch__occupancy_limit_shared_mem", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "lts__t_bytes.sum",
]


def summarise(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for vals in rows[2:]:
        d = {"kernel": vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else ""}
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                d[k] = f"{vals[i]} {units[i]}".strip()
        stalls = []
        for i, h in enumerate(hdr):
            if h.startswith("smsp__average_warp_latency_issue_stalled_") and h.endswith(".ratio") or \
               (h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("_not_issued")):
                try:
                    stalls.append((float(vals[i]), h))
                except ValueError:
                    pass
        stalls.sort(reverse=True)
        d["top_stalls"] = [f"{h.split('stalled_')[-1]}={v:g}" for v, h in stalls[:8]]
        res.append(d)
    return res


if __name__ == "__main__":
    out = []
    for path in sys.argv[1:]:
        out.extend(summarise(path))
    print(json.dumps(out, indent=1))
