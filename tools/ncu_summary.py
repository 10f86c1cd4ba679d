"""Summarise an ncu report (details page + SASS hot spots) — run here, no GPU."""
import collections, csv, io, subprocess, sys

rep = sys.argv[1]
keys = ["Duration", "DRAM Throughput", "Memory Throughput", "L1/TEX Cache Throughput", "L2 Cache Throughput",
        "Compute (SM) Throughput", "Executed Ipc Active", "Issue Slots Busy", "Registers Per Thread",
        "Achieved Occupancy", "Theoretical Occupancy", "Warp Cycles Per Issued Instruction", "Issued Instructions",
        "Dynamic Shared Memory Per Block", "Grid Size", "Block Limit Registers", "Block Limit Shared Mem",
        "L1/TEX Hit Rate", "L2 Hit Rate", "Eligible Warps Per Scheduler", "No Eligible"]
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
for row in csv.DictReader(io.StringIO(out)):
    if row.get("Metric Name") in keys:
        print(f"{row['Metric Name']:<40} {row['Metric Value']} {row['Metric Unit']}")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
if len(rows) > 2:
    hdr, units, vals = rows[0], rows[1], rows[2]
    for k in ("dram__bytes_read.sum", "dram__bytes_write.sum", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
              "smsp__inst_executed_pipe_fp64.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
              "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"):
        if k in hdr:
            i = hdr.index(k)
            print(f"{k:<60} {vals[i]} {units[i]}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
srows = list(csv.reader(io.StringIO(src)))
if len(srows) > 2:
    hdr = srows[1]
    ix = {h: i for i, h in enumerate(hdr)}
    by = collections.Counter(); st = collections.Counter()
    for r in srows[2:]:
        if len(r) <= max(ix["Source"], ix["Instructions Executed"], ix["Warp Stall Sampling (All Samples)"]):
            continue
        s = r[ix["Source"]].strip()
        toks = s.split()
        if not toks:
            continue
        op = (toks[1] if toks[0].startswith("@") else toks[0]).split(".")[0]
        if not r[ix["Instructions Executed"]].strip().isdigit():
            continue
        by[op] += int(r[ix["Instructions Executed"]] or 0)
        st[op] += int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    tot = sum(by.values()) or 1
    print("opcode mix (warp instructions executed, stall samples):")
    for op, c in by.most_common(14):
        print(f"  {op:<8} {c:>12} {100 * c / tot:5.1f}%  stalls {st[op]}")
    print("top stall sites:")
    good = [r for r in srows[2:] if len(r) > ix["Warp Stall Sampling (All Samples)"]
            and r[ix["Warp Stall Sampling (All Samples)"]].strip().isdigit()]
    for r in sorted(good, key=lambda r: -int(r[ix["Warp Stall Sampling (All Samples)"]] or 0))[:16]:
        print("  ", r[ix["Source"]][:70].ljust(70), r[ix["Warp Stall Sampling (All Samples)"]])
