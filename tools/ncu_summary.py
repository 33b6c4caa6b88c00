"""Summarise an ncu report: key metrics + per-source-line instruction/stall hot spots."""
import collections, csv, io, subprocess, sys
rep = sys.argv[1]
def run(*a):
    return subprocess.run(["ncu", "-i", rep, *a], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(run("--page", "raw", "--csv"))))
h, v = r[0], r[2]
keys = ["gpu__time_duration.sum", "sm__cycles_active.max", "sm__cycles_active.avg", "smsp__inst_executed.sum",
        "launch__grid_size", "launch__block_size", "launch__registers_per_thread", "dram__bytes_read.sum",
        "dram__bytes_write.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed_pipe_fp64.sum",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active"]
for i, n in enumerate(h):
    if n in keys:
        print(f"{n:55s} {v[i]}")
stalls = []
for i, n in enumerate(h):
    if n.startswith("smsp__pcsamp_warps_issue_stalled_") and not n.endswith("_not_issued"):
        try: stalls.append((float(v[i].replace(",", "")), n[len("smsp__pcsamp_warps_issue_stalled_"):]))
        except ValueError: pass
ts = sum(x[0] for x in stalls) or 1.0
print("stall reasons (pc samples): " + ", ".join(f"{n} {100 * c / ts:.1f}%" for c, n in sorted(stalls, reverse=True)[:8]))
for i, n in enumerate(h):
    if n in ("smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
             "l1tex__data_pipe_lsu_wavefronts_mem_shared.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed_pipe_lsu.sum",
             "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
             "lts__t_sector_hit_rate.pct"):
        print(f"{n:55s} {v[i]}")
rows = list(csv.reader(io.StringIO(run("--page", "source", "--csv", "--print-source", "cuda,sass"))))
agg = collections.defaultdict(lambda: [0, 0]); cur = None; fname = None; hdr = None
for row in rows:
    if row and row[0] == "File Path": fname = row[1].split("/")[-1]; continue
    if row and row[0] == "Line No": hdr = row; continue
    if not hdr or len(row) < 8: continue
    if row[0]: cur = (fname, row[0], row[1].strip()[:80])
    try: agg[cur][0] += int(row[7] or 0); agg[cur][1] += int(row[4] or 0)
    except ValueError: pass
tot = sum(x[0] for x in agg.values()); tots = sum(x[1] for x in agg.values())
print(f"warp instructions {tot}  stall samples {tots}")
for k, x in sorted(agg.items(), key=lambda kv: -kv[1][1])[: int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    print(f"{x[0]:9d} {x[1]:5d}  {k[0]}:{k[1]}  {k[2]}")
