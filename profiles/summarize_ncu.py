"""Summarise ncu reports (.ncu-rep) into profiles/ncu_summary.json + a
markdown table.  Run here (no GPU needed):

    python profiles/summarize_ncu.py <tag> <kernel_key> <s> <report.ncu-rep> [...]

kernel_key names the kernel in the summary (e.g. sys_attn_sm100_kernel), or
"auto" to key every kernel of the report by its own name; s is the
system-prompt length of the bench workload the capture came from.
"""

import csv
import io
import json
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_tensor_subpipe_hmma.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "lts__t_sector_hit_rate.pct",
    # tcgen05 (UTC*MMA) and legacy HMMA activity of the tensor pipe, the
    # SFU (MUFU.EX2) pipe, and the warp stall breakdown per issued instruction
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_branch_resolving_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_selected_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_sleeping_per_issue_active.ratio",
    # tcgen05 evidence: UTCHMMA instructions (the hmma subpipe counts
    # HMMA/UTCHMMA/UTCQMMA/UTCOMMA), tensor-memory activity, shared-memory
    # wavefronts feeding the tensor core, and the SM clock the kernel ran at
    "sm__inst_executed_pipe_tensor_subpipe_hmma.sum",
    "sm__pipe_tensor_subpipe_hmma_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_xu_realtime.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_tmem.avg.pct_of_peak_sustained_active",
    "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_tc_wavefronts_mem_shared.sum",
    "sm__cycles_elapsed.avg.per_second",
]
SCALE = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1.0, "us": 1e-6, "ns": 1e-9,
         "ms": 1e-3, "msecond": 1e-3, "usecond": 1e-6, "nsecond": 1e-9}


def read(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    # triage metrics carry a section prefix ("TPC.TriageCompute.<metric>")
    hdr = [h.split("TriageCompute.", 1)[1] if "TriageCompute." in h else h for h in rows[0]]
    units = rows[1]
    res = []
    for vals in rows[2:]:
        rec = {"kernel": vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else ""}
        for m in METRICS:
            if m in hdr:
                i = hdr.index(m)
                try:
                    v = float(vals[i].replace(",", ""))
                except ValueError:
                    continue
                u = units[i]
                if u in SCALE:
                    v *= SCALE[u]
                    u = "s" if u.endswith("s") or "second" in u else "bytes"
                rec[m] = v
        res.append(rec)
    return res


def main():
    tag, key, s = sys.argv[1], sys.argv[2], sys.argv[3]
    path = os.path.join(HERE, "ncu_summary.json")
    data = json.load(open(path)) if os.path.exists(path) else {"kernels": {}}
    for rep in sys.argv[4:]:
        for rec in read(rep):
            rec["dram_bytes"] = rec.get("dram__bytes_read.sum", 0) + rec.get("dram__bytes_write.sum", 0)
            rec["report"] = os.path.basename(rep)
            rec["tag"] = tag
            k = key
            if key == "auto":
                name = rec["kernel"].split("(")[0].split("<")[0].strip()
                k = name.split()[-1].split("::")[-1]
            data["kernels"].setdefault(k, {})[str(s)] = rec
            print(json.dumps(rec, indent=1))
    json.dump(data, open(path, "w"), indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
