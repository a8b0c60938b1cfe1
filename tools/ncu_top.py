"""Summarise an ncu report: stall reasons and top SASS lines (debug aid).
usage: python tools/ncu_top.py report.ncu-rep [N]"""
import csv, io, subprocess, sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 20
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, vals = rows[0], rows[2]
want = ["gpu__time_duration.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__inst_executed.avg.per_cycle_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__registers_per_thread",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__cycles_active.avg"]
for h, v in zip(hdr, vals):
    if h in want or ("pcsamp_warps_issue_stalled" in h and not h.endswith("not_issued")
                     and v.replace(".", "").isdigit() and float(v) > 1000):
        print(f"{h:70s} {v}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hdr, data = rows[1], rows[2:]
i_s, i_src, i_ex = (hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Source"),
                    hdr.index("Instructions Executed"))
stall = [j for j, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
print("samples", sum(int(r[i_s]) for r in data))
for r in sorted(data, key=lambda r: -int(r[i_s]))[:n]:
    st = sorted(((int(r[j]) if r[j].isdigit() else 0, hdr[j]) for j in stall), reverse=True)[:2]
    print(r[i_s], r[i_ex], r[i_src].strip()[:64], st)
