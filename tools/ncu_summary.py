"""Summaries of ncu output for profiles/: per-kernel launch aggregation of a
`--metrics gpu__time_duration.sum` CSV and key metrics of a `--set full` report."""
import collections
import csv
import io
import subprocess
import sys


def launches(path):
    lines = open(path).read().splitlines()
    start = [i for i, l in enumerate(lines) if l.startswith('"ID"')][0]
    rows = list(csv.DictReader(io.StringIO("\n".join(lines[start:]))))
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows:
        n = r["Kernel Name"].split("(")[0]
        agg[n][0] += 1
        agg[n][1] += float(r["Metric Value"].replace(",", ""))
    # bench.py holds the GPU with torch's spin kernel (torch.cuda._sleep) while it enqueues
    # the timed steps: idle time, not work -- listed, but outside the shares
    idle = {n for n in agg if "spin_kernel" in n}
    tot = sum(v[1] for n, v in agg.items() if n not in idle)
    out = [f"# {path}: {len(rows)} launches, gpu__time_duration.sum (ns), cold-cache serialised (ncu); "
           f"shares exclude the host-enqueue spin kernel",
           f"{'kernel':64s} {'launches':>8s} {'total_us':>10s} {'us/launch':>10s} {'share':>6s}"]
    for n, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        share = "  idle" if n in idle else f"{100 * t / tot:5.1f}%"
        out.append(f"{n[:64]:64s} {c:8d} {t / 1e3:10.1f} {t / c / 1e3:10.2f} {share}")
    return "\n".join(out)


KEYS = ["Duration", "Compute (SM) Throughput", "Memory Throughput", "DRAM Throughput", "L2 Cache Throughput",
        "Issue Slots Busy", "Executed Ipc Active", "Registers Per Thread", "Grid Size", "Block Size",
        "Achieved Occupancy", "Eligible Warps Per Scheduler", "L2 Hit Rate", "Dynamic Shared Memory Per Block"]
RAW = ["dram__bytes_read.sum", "dram__bytes_write.sum",
       "sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32_sparsity_off.sum.pct_of_peak_sustained_elapsed",
       "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
       "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
       "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
       "gpu__time_duration.sum"]


def full(path):
    det = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(det)))
    h = r[0]
    out = [f"# {path} (ncu --set full)"]
    seen = set()
    for row in r[1:]:
        d = dict(zip(h, row))
        if d.get("Metric Name") in KEYS and (d["ID"], d["Metric Name"]) not in seen:
            seen.add((d["ID"], d["Metric Name"]))
            out.append(f"[{d['ID']}] {d['Kernel Name'][:50]:50s} {d['Metric Name']:36s} {d['Metric Value']} {d['Metric Unit']}")
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    if len(rr) > 2:
        hh, uu = rr[0], rr[1]
        for i, row in enumerate(rr[2:]):
            for k, u, v in zip(hh, uu, row):
                if k in RAW:
                    out.append(f"[{i}] raw {k} = {v} {u}")
    return "\n".join(out)


if __name__ == "__main__":
    kind, path = sys.argv[1], sys.argv[2]
    print(launches(path) if kind == "launches" else full(path))
