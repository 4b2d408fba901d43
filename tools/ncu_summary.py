"""Summarise an `ncu --set full` report: per launch, the metrics DESIGN.md and
profiles/ quote (DRAM bytes, duration, achieved GB/s, SMEM wavefronts per record,
issue activity, warp stalls).  Usage: python tools/ncu_summary.py rep.ncu-rep records_per_launch,..."""
import csv, io, subprocess, sys

M = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
     "lts__t_requests_srcunit_tex_op_write.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
     "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__inst_executed.sum",
     "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
     "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
     "launch__shared_mem_per_block_dynamic",
     "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
     "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
     "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
     "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
     "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio"]
rep = sys.argv[1]
recs = [float(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else []
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(M)],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, units = rows[0], rows[1]
unit_scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3,
              "ns": 1e-9, "us": 1e-6, "ms": 1e-3}
for li, r in enumerate(rows[2:]):
    d = dict(zip(hdr, r)); u = dict(zip(hdr, units))
    def val(m):
        v = float(d[m].replace(",", ""))
        return v * unit_scale.get(u[m], 1)
    name = d["Kernel Name"].split("(")[0]
    t = val("gpu__time_duration.sum"); rd = val("dram__bytes_read.sum"); wr = val("dram__bytes_write.sum")
    n = recs[li] if li < len(recs) else None
    print(f"{name}  (launch {li})")
    for m in M:
        print(f"    {m:80s} {d[m]:>16s} {u[m]}")
    line = f"    => dram {(rd + wr) / 1e9:.2f} GB in {t * 1e3:.3f} ms = {(rd + wr) / t / 1e12:.2f} TB/s"
    if n:
        line += (f"; {(rd + wr) / n:.2f} B/record; "
                 f"{val('l1tex__data_pipe_lsu_wavefronts_mem_shared.sum') / n:.2f} SMEM wavefronts/record; "
                 f"{val('smsp__inst_executed.sum') / n:.2f} warp-inst/record")
    print(line + "\n")
