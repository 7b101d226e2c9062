"""Summarise an ncu report (raw page) into the JSON kept under profiles/.
Usage: python tools/ncu_summary.py REPORT.ncu-rep OUT.json [kernel-regex]"""
import csv, io, json, subprocess, sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "l1tex__lsu_writeback_active.avg.pct_of_peak_sustained_elapsed",
    "lts__t_bytes.sum", "smsp__warps_active.avg.per_cycle_active", "smsp__warps_eligible.avg.per_cycle_active",
    "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic", "launch__grid_size",
    "launch__block_size", "sm__cycles_elapsed.avg.per_second",
]


def main():
    rep, out = sys.argv[1], sys.argv[2]
    cmd = ["ncu", "-i", rep, "--page", "raw", "--csv"]
    if len(sys.argv) > 3:
        cmd += ["-k", "regex:" + sys.argv[3]]
    txt = subprocess.run(cmd, capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = dict(zip(hdr, vals))
    u = dict(zip(hdr, units))
    res = {"kernel": d.get("Kernel Name", "")}
    for k in KEYS:
        if k in d:
            res[k] = f"{d[k]} {u.get(k, '')}".strip()
    stalls = {}
    for k, v in d.items():
        if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
            try:
                stalls[k[len("smsp__pcsamp_warps_issue_stalled_"):]] = int(float(v))
            except ValueError:
                pass
    res["stall_samples"] = stalls
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
