"""Summarise an ncu report into a small text file for profiles/.

    python tools/ncu_summary.py report.ncu-rep [title] > profiles/rNN_name.txt
"""
import csv
import io
import subprocess
import sys

KEYS = ["Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput", "Executed Ipc Active",
        "Issue Slots Busy", "Warp Cycles Per Issued Instruction", "Registers Per Thread", "Achieved Occupancy",
        "Theoretical Occupancy", "Executed Instructions", "L2 Hit Rate", "L1/TEX Hit Rate", "Block Size", "Grid Size",
        "Dynamic Shared Memory Per Block", "SM Frequency", "DRAM Frequency"]
RAW = ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum", "sm__inst_executed.sum",
       "smsp__inst_executed_op_shared_ld.sum", "sm__sass_thread_inst_executed_op_dfma_pred_on.sum",
       "sm__sass_thread_inst_executed_op_dadd_pred_on.sum", "sm__sass_thread_inst_executed_op_dmul_pred_on.sum"]


def ncu(args):
    return subprocess.run(["ncu"] + args, capture_output=True, text=True).stdout


def main(rep, title=""):
    print(f"# ncu summary: {title or rep}")
    det = list(csv.reader(io.StringIO(ncu(["-i", rep, "--page", "details", "--csv"]))))
    hdr = det[0]
    iname = hdr.index("Kernel Name")
    imet, iunit, ival = hdr.index("Metric Name"), hdr.index("Metric Unit"), hdr.index("Metric Value")
    seen = set()
    kern = None
    for r in det[1:]:
        if len(r) <= ival:
            continue
        kern = r[iname]
        if r[imet] in KEYS and r[imet] not in seen:
            seen.add(r[imet])
            print(f"{r[imet]:40s} {r[ival]:>16s} {r[iunit]}")
    print(f"kernel: {kern}")
    raw = list(csv.reader(io.StringIO(ncu(["-i", rep, "--page", "raw", "--csv"]))))
    if len(raw) >= 3:
        h, u, v = raw[0], raw[1], raw[2]
        for k in RAW:
            if k in h:
                i = h.index(k)
                print(f"{k:40s} {v[i]:>16s} {u[i]}")
    src = ncu(["-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"])
    rows = []
    cur = "?"
    for r in csv.reader(io.StringIO(src)):
        if len(r) >= 2 and r[0] in ("File Path", "File Name"):
            cur = r[1].split("/")[-1]
            continue
        if len(r) > 6 and r[0] not in ("", "Line No"):
            try:
                s = int(r[4])
            except ValueError:
                continue
            if s:
                rows.append((s, cur, r[0], r[1].strip()[:90]))
    tot = sum(x[0] for x in rows) or 1
    rows.sort(reverse=True)
    print("\n## warp-stall samples by source line (top 15)")
    for s, fn, ln, text in rows[:15]:
        print(f"{100.0 * s / tot:5.1f}%  {fn}:{ln}  {text}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "")
