"""Summarise ncu reports (--page raw) into the JSON kept under profiles/:
per launch the duration, DRAM bytes, issue / LSU utilisation, shared-memory
wavefronts and bank conflicts, tensor-pipe activity and the top warp-stall
reasons. Usage: python tools/ncu_summary.py OUT.json name=REPORT.ncu-rep ..."""
import csv
import io
import json
import subprocess
import sys

KEYS = {
    "duration_us": "gpu__time_duration.sum",
    "dram_read_bytes": "dram__bytes_read.sum",
    "dram_write_bytes": "dram__bytes_write.sum",
    "issue_active_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "lsu_wavefronts_pct": "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
    "shared_wavefronts": "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "shared_bank_conflicts": "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "tensor_pipe_active_pct": "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active",
    "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "dram_throughput_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "registers": "launch__registers_per_thread",
    "inst_executed": "smsp__inst_executed.sum",
    "thread_inst_per_inst": "smsp__thread_inst_executed_per_inst_executed.ratio",
    "grid": "launch__grid_size",
    "block": "launch__block_size",
}
SCALE = {"dram__bytes_read.sum": None, "dram__bytes_write.sum": None}


def raw(report):
    out = subprocess.run(["ncu", "-i", report, "--page", "raw", "--csv", "--print-units", "base"],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[2:]


def summarise(report):
    hdr, rows = raw(report)
    res = []
    for v in rows:
        d = dict(zip(hdr, v))
        e = {"kernel": d.get("Kernel Name", "")}
        for k, m in KEYS.items():
            try:
                e[k] = float(d[m].replace(",", ""))
            except (KeyError, ValueError):
                e[k] = None
        if e["duration_us"] is not None:
            e["duration_us"] /= 1e3  # base unit ns
        stalls = {}
        for k, x in d.items():
            if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
                try:
                    stalls[k[len("smsp__pcsamp_warps_issue_stalled_"):]] = float(x.replace(",", ""))
                except ValueError:
                    pass
        tot = sum(stalls.values()) or 1.0
        e["top_stalls_pct"] = {k: round(100 * v / tot, 1) for k, v in sorted(stalls.items(), key=lambda kv: -kv[1])[:6]}
        res.append(e)
    return res


def main():
    out = {}
    for arg in sys.argv[2:]:
        name, rep = arg.split("=", 1)
        out[name] = summarise(rep)
    with open(sys.argv[1], "w") as fh:
        json.dump(out, fh, indent=1)
    print(json.dumps({k: [(e["kernel"][:40], e["duration_us"]) for e in v] for k, v in out.items()}, indent=1))


if __name__ == "__main__":
    main()
