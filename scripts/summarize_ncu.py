"""Summarise an ncu launch-list CSV (gpu__time_duration + dram bytes per launch)
and an ncu --set full report into profiles/ text files."""
import collections
import csv
import subprocess
import sys


def launches(path):
    rows = list(csv.reader(l for l in open(path) if l.startswith('"')))
    hdr, rows = rows[0], rows[1:]
    K, M, V, I = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
    d = collections.defaultdict(dict)
    for r in rows:
        d[int(r[I])][r[M]] = float(r[V].replace(",", ""))
        d[int(r[I])]["k"] = r[K].split("(")[0].replace("void ", "")
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0, 0.0])
    for x in d.values():
        a = agg[x["k"]]
        a[0] += 1
        a[1] += x.get("gpu__time_duration.sum", 0)
        a[2] += x.get("dram__bytes_read.sum", 0)
        a[3] += x.get("dram__bytes_write.sum", 0)
    tot = sum(a[1] for a in agg.values())
    out = [f"# {path}: {len(d)} launches, total device time {tot / 1e6:.3f} ms (ncu: cold-cache, serialised)",
           f"{'kernel':40s} {'launches':>8s} {'avg_us':>9s} {'share':>7s} {'dram_rd_MB':>11s} {'dram_wr_MB':>11s} {'GB/s':>8s}"]
    for k, a in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        n = a[0]
        out.append(f"{k:40s} {n:8d} {a[1] / n / 1e3:9.1f} {a[1] / tot:7.3f} {a[2] / n / 1e6:11.1f} {a[3] / n / 1e6:11.1f}"
                   f" {(a[2] + a[3]) / a[1]:8.1f}")
    return "\n".join(out)


def full(path):
    res = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(res.splitlines()))
    h = rows[0]
    ki, si, mi, vi, ui = (h.index(k) for k in ("Kernel Name", "Section Name", "Metric Name", "Metric Value",
                                                 "Metric Unit"))
    out = [f"# ncu --set full: {path}"]
    last = None
    for r in rows[1:]:
        k = r[ki].split("(")[0]
        if k != last:
            out.append(f"\n## {k}")
            last = k
        out.append(f"{r[si][:28]:28s} {r[mi][:44]:44s} {r[vi]:>14s} {r[ui]}")
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(raw.splitlines()))
    hh = rr[0]
    want = ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum", "launch__registers_per_thread",
            "sm__warps_active.avg.pct_of_peak_sustained_active", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
            "lts__t_bytes.sum", "smsp__inst_executed.sum"]
    out.append("\n## raw metrics per profiled launch")
    for r in rr[2:]:
        out.append(r[hh.index("Kernel Name")].split("(")[0] + ": " +
                   ", ".join(f"{w}={r[hh.index(w)]}" for w in want if w in hh))
    return "\n".join(out)


if __name__ == "__main__":
    kind, src, dst = sys.argv[1:4]
    txt = launches(src) if kind == "launches" else full(src)
    open(dst, "w").write(txt + "\n")
    print(txt[:3000])
