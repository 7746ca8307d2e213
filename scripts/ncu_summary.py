"""Summarise one `ncu --set full` report: key metrics, stall reasons and the
hottest source lines of every kernel in it.
  python scripts/ncu_summary.py <report.ncu-rep> <title> [out.txt]"""
import csv, subprocess, sys

rep, title = sys.argv[1], sys.argv[2]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(raw.splitlines()))
H, U = r[0], r[1]
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "launch__occupancy_limit_registers", "sm__cycles_elapsed.avg",
        "l1tex__t_bytes_pipe_lsu_mem_local_op_ld.sum", "l1tex__t_bytes_pipe_lsu_mem_local_op_st.sum"]
lines = [title, ""]
for V in r[2:]:
    m = {H[i]: (V[i], U[i]) for i in range(len(H))}
    lines.append(f"== {m.get('Kernel Name', ('?',))[0][:110]}")
    for k in keys:
        if k in m:
            lines.append(f"  {k:70s} {m[k][0]:>16s} {m[k][1]}")
    st = []
    for k, (v, u) in m.items():
        if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
            try:
                st.append((float(v), k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
            except ValueError:
                pass
    lines += ["  warp stall reasons (warps stalled per issue-active cycle):"]
    lines += [f"    {x:6.2f} {n}" for x, n in sorted(st, reverse=True)[:8]]
    lines.append("")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
cur, fn, hot = None, None, {}
for x in csv.reader(src.splitlines()):
    if len(x) >= 2 and x[0] == "File Path":
        cur = x[1].split("/")[-1]
    elif len(x) >= 2 and x[0] == "Function Name":
        fn = x[1]
    elif len(x) > 6 and x[0].isdigit() and x[2] == "-":
        try:
            hot.setdefault(fn, []).append((float(x[4]), float(x[7] or 0), cur, int(x[0]), x[1].strip()[:90]))
        except ValueError:
            pass
for fn, h in hot.items():
    tot = sum(q[0] for q in h) or 1
    lines += ["", f"hottest source lines of {fn[:100]} (share of warp stall samples, instructions executed):"]
    for s_, n_, f_, l_, t_ in sorted(h, reverse=True)[:25]:
        lines.append(f"  {100 * s_ / tot:5.1f}% {n_:10.0f}  {f_}:{l_}  {t_}")
text = "\n".join(lines) + "\n"
if len(sys.argv) > 3:
    open(sys.argv[3], "w").write(text)
print(text)
