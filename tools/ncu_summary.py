"""Summarise ncu outputs for profiles/: a launch list CSV (gpu__time_duration.sum per
launch) into per-kernel shares, and a `--page raw --csv` export into key metrics."""
import collections
import csv
import sys

KEY = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
       "lts__t_sectors_srcunit_tex_op_read.sum", "lts__t_sector_hit_rate.pct",
       "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
       "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum", "l1tex__t_sector_hit_rate.pct",
       "sm__throughput.avg.pct_of_peak_sustained_elapsed",
       "lts__throughput.avg.pct_of_peak_sustained_elapsed",
       "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
       "dram__throughput.avg.pct_of_peak_sustained_elapsed",
       "sm__warps_active.avg.pct_of_peak_sustained_active",
       "smsp__issue_active.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
       "smsp__inst_executed.sum", "launch__registers_per_thread", "launch__grid_size",
       "launch__block_size", "launch__occupancy_limit_registers",
       "sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_uniform.avg.pct_of_peak_sustained_active",
       "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed",
       "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
       "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
       "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
       "launch__occupancy_limit_shared_mem",
       "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
       "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
       "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
       "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio"]

SCALE = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6, "s": 1e6}


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    mi = h.index("Metric Name") if "Metric Name" in h else None
    tot, cnt = collections.defaultdict(float), collections.Counter()
    dram = collections.defaultdict(float)
    for r in rows[hdr + 1:]:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0].replace("void ", "")[:70]
        metric = r[mi] if mi is not None else "gpu__time_duration.sum"
        if metric.startswith("dram__bytes"):  # captured alongside: bytes per kernel
            dram[name] += float(r[vi].replace(",", "")) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6,
                                                           "Gbyte": 1e9}.get(r[ui], 1.0)
            continue
        if metric != "gpu__time_duration.sum":
            continue
        us = float(r[vi].replace(",", "")) * SCALE.get(r[ui], 1.0)
        tot[name] += us
        cnt[name] += 1
    T = sum(tot.values())
    if dram:
        out = ["| kernel | launches | total µs | share | DRAM MB |", "|---|---:|---:|---:|---:|"]
        for k, v in sorted(tot.items(), key=lambda x: -x[1]):
            out.append(f"| `{k}` | {cnt[k]} | {v:,.0f} | {100 * v / T:.1f}% | {dram[k] / 1e6:,.0f} |")
    else:
        out = ["| kernel | launches | total µs | share |", "|---|---:|---:|---:|"]
        for k, v in sorted(tot.items(), key=lambda x: -x[1]):
            out.append(f"| `{k}` | {cnt[k]} | {v:,.0f} | {100 * v / T:.1f}% |")
    return "\n".join(out)


def raw(path):
    rows = list(csv.reader(open(path)))
    h, units = rows[0], rows[1]
    out = []
    for n, r in enumerate(rows[2:]):
        name = r[h.index("Kernel Name")] if "Kernel Name" in h else "?"
        out.append(f"\n**launch {n}: `{name.split('(')[0]}`**\n\n| metric | value | unit |\n|---|---:|---|")
        for k in KEY:
            if k in h:
                i = h.index(k)
                out.append(f"| {k} | {r[i]} | {units[i]} |")
    return "\n".join(out)


if __name__ == "__main__":
    kind, path = sys.argv[1], sys.argv[2]
    print(launches(path) if kind == "launches" else raw(path))
