"""Summarise ncu artefacts into profiles/ (launch-list shares + key metrics of
the top kernels).  Usage: python tools/summarize_profile.py <launches.csv> <report.ncu-rep>..."""
import collections
import csv
import subprocess
import sys


def launch_shares(path, last_fraction=0.5, last_n=None):
    rows = list(csv.reader(open(path)))
    hdr = None
    data = []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    data = data[-last_n:] if last_n else data[int(len(data) * (1 - last_fraction)):]
    agg = collections.defaultdict(lambda: [0, 0.0])
    for d in data:
        name = d["Kernel Name"].split("(")[0].replace("void ", "").replace("(anonymous namespace)::", "")
        v = float(d["Metric Value"].replace(",", ""))
        unit = d["Metric Unit"]
        v *= {"msecond": 1e6, "usecond": 1e3, "nsecond": 1.0, "second": 1e9}.get(unit, 1.0)
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(v[1] for v in agg.values())
    what = f"last {last_n} launches" if last_n else f"last {int(last_fraction*100)}% of launches"
    out = [f"launch list (ncu gpu__time_duration.sum, --clock-control none; {what} = one step)",
           f"{'kernel':58s} {'launches':>8s} {'ms':>10s} {'share':>7s}"]
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])[:20]:
        out.append(f"{k[:58]:58s} {v[0]:8d} {v[1] / 1e6:10.2f} {100 * v[1] / tot:6.2f}%")
    out.append(f"total {tot / 1e6:.1f} ms over {sum(v[0] for v in agg.values())} launches")
    return "\n".join(out)


WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "sm__cycles_elapsed.avg.per_second",
        "smsp__pcsamp_warps_issue_stalled_long_scoreboard", "smsp__pcsamp_warps_issue_stalled_wait",
        "smsp__pcsamp_warps_issue_stalled_barrier", "smsp__pcsamp_warps_issue_stalled_short_scoreboard"]


def report_metrics(path):
    txt = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    hdr, units = rows[0], rows[1]
    out = []
    for vals in rows[2:]:
        name = vals[hdr.index("Kernel Name")]
        out.append(f"kernel: {name[:110]}")
        for w in WANT:
            for i, h in enumerate(hdr):
                if h == w or h.endswith("." + w):
                    out.append(f"  {w} = {vals[i]} {units[i]}")
                    break
    return "\n".join(out)


if __name__ == "__main__":
    args = sys.argv[1:]
    last_n = None
    if args and args[0].startswith("--last="):
        last_n = int(args.pop(0).split("=")[1])
    print(launch_shares(args[0], last_n=last_n))
    for p in args[1:]:
        print()
        print(report_metrics(p))
