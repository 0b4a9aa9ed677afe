"""Summarise an ncu report: key raw metrics + top SASS lines by stall samples."""
import csv, subprocess, sys, io
rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__thread_inst_executed_per_inst_executed.ratio", "smsp__inst_executed.sum", "launch__registers_per_thread",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem", "sm__maximum_warps_per_active_cycle_pct",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "launch__grid_size", "launch__block_size",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct"]
for r in rows[2:]:
    d = dict(zip(hdr, r))
    print(d.get("Kernel Name", "")[:90])
    for k in keys:
        if k in d:
            print("  %-66s %s %s" % (k, d[k], units[hdr.index(k)]))
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hdr = rows[1]; idx = {h: i for i, h in enumerate(hdr)}
data = [r for r in rows[2:] if len(r) == len(hdr)]
ts = sum(float(r[idx["Warp Stall Sampling (All Samples)"]] or 0) for r in data) or 1
ti = sum(float(r[idx["Instructions Executed"]] or 0) for r in data)
print("total warp-inst %.3e  samples %d" % (ti, ts))
for r in sorted(data, key=lambda r: -float(r[idx["Warp Stall Sampling (All Samples)"]] or 0))[:top]:
    print("%6.1f%% %9.1fM  %s" % (100 * float(r[idx["Warp Stall Sampling (All Samples)"]] or 0) / ts,
                                 float(r[idx["Instructions Executed"]] or 0) / 1e6, r[idx["Source"]][:80]))
