"""Summarises ncu --set full reports (raw page) into one JSON object per kernel:
duration, SM clock, tensor-pipe / DRAM / smem utilisation and DRAM bytes.  Usage:
  python scripts/ncu_summary.py gpurun_out/prof_gemm.ncu-rep [...] > profiles/rNN/ncu_summary.json"""
import csv
import io
import json
import subprocess
import sys

KEYS = {
    "duration_us": "gpu__time_duration.sum",
    "sm_freq_ghz": "smsp__cycles_elapsed.avg.per_second",
    "tc_pipe_active_pct_elapsed": "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "tc_pipe_active_pct_active": "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active",
    "utchmma_bf16_pct_peak": "sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32_sparsity_off.avg.pct_of_peak_sustained_elapsed",
    "hmma_bf16_pct_peak": "sm__ops_path_tensor_op_hmma_src_bf16_dst_fp32_sparsity_off.avg.pct_of_peak_sustained_elapsed",
    "dram_read_bytes": "dram__bytes_read.sum",
    "dram_write_bytes": "dram__bytes_write.sum",
    "dram_throughput_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm_throughput_pct": "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "smem_tc_wavefronts_pct": "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "xu_mufu_pipe_pct_active": "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "issue_active_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "registers": "launch__registers_per_thread",
    "grid": "launch__grid_size",
    "block": "launch__block_size",
}
SCALE = {"ms": 1e3, "us": 1.0, "ns": 1e-3, "Mbyte": 1e6, "Kbyte": 1e3, "Gbyte": 1e9, "byte": 1.0, "usecond": 1.0, "msecond": 1e3, "nsecond": 1e-3,
         "Ghz": 1.0, "cycle/nsecond": 1.0, "cycle/usecond": 1e-3}


def summarise(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        rec = {"kernel": d.get("Kernel Name", "")[:120], "report": path}
        for k, m in KEYS.items():
            if m in d and d[m] not in ("", "n/a"):
                try:
                    v = float(d[m].replace(",", ""))
                except ValueError:
                    continue
                u = units[hdr.index(m)]
                rec[k] = v * SCALE.get(u, 1.0)
        if "dram_read_bytes" in rec and "dram_write_bytes" in rec:
            rec["dram_traffic_bytes"] = rec["dram_read_bytes"] + rec["dram_write_bytes"]
        out.append(rec)
    return out


if __name__ == "__main__":
    res = []
    for p in sys.argv[1:]:
        res.extend(summarise(p))
    print(json.dumps(res, indent=1))
