"""Summarise an ncu report: key SOL metrics, instruction mix and top stall reasons per opcode.
python tools/ncu_summary.py gpurun_out/x.ncu-rep [--json out.json]"""
import collections
import csv
import io
import json
import subprocess
import sys

rep = sys.argv[1]


def ncu(*a):
    return subprocess.run(["ncu", "-i", rep, *a], capture_output=True, text=True).stdout


raw = list(csv.reader(io.StringIO(ncu("--page", "raw", "--csv"))))
hdr, units, vals = raw[0], raw[1], raw[2]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "smsp__inst_executed.avg.per_cycle_active", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_bytes.sum", "launch__grid_size", "launch__block_size", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.sum", "smsp__average_warp_latency_issue_stalled_barrier",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]
out = {}
for w in want:
    if w in hdr:
        i = hdr.index(w)
        out[w] = (vals[i], units[i])
for k, (v, u) in out.items():
    print(f"{k:70s} {v} {u}")
src = list(csv.reader(io.StringIO(ncu("--page", "source", "--csv", "--print-source", "sass"))))
h = src[1]
ie, sc = h.index("Instructions Executed"), h.index("Source")
stc = [i for i, c in enumerate(h) if c.startswith("stall_")] if False else []
st = h.index("Warp Stall Sampling (All Samples)")
op, stall, tot, tst = collections.Counter(), collections.Counter(), 0.0, 0.0
for x in src[2:]:
    try:
        n, s = float(x[ie] or 0), float(x[st] or 0)
    except (ValueError, IndexError):
        continue
    t = x[sc].strip().split()
    if not t:
        continue
    o = t[1] if t[0].startswith("@") else t[0]
    o = o.split(".")[0]
    op[o] += n
    stall[o] += s
    tot += n
    tst += s
print(f"total warp instructions {tot:.4g}")
for o, n in op.most_common(18):
    print(f"  {o:10s} {n / tot * 100:6.2f}% inst {stall[o] / max(tst, 1) * 100:6.2f}% stall-samples")
# stall reasons (summed over the kernel)
det = list(csv.reader(io.StringIO(ncu("--page", "details", "--csv", "--section", "WarpStateStats"))))
for row in det[1:]:
    if len(row) > 14 and "Stall" in row[12]:
        pass
if "--json" in sys.argv:
    json.dump({k: v for k, (v, u) in out.items()}, open(sys.argv[sys.argv.index("--json") + 1], "w"), indent=1)
