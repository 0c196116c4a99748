"""Summarise an ncu --csv launch list (dev tool): per launch duration, DRAM GB, DMMA-active %."""
import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hdr]
K, M, V, I, G = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "ID", "Grid Size"))
d, names = collections.defaultdict(dict), {}
for r in rows[hdr + 1:]:
    if len(r) < len(h):
        continue
    d[r[I]][r[M]] = float(r[V].replace(",", ""))
    names[r[I]] = (r[K].split("(")[0][-34:], r[G])
tot = 0.0
for i in sorted(d, key=int):
    x = d[i]
    t = x.get("gpu__time_duration.sum", 0) / 1e3
    tot += t
    gb = (x.get("dram__bytes_read.sum", 0) + x.get("dram__bytes_write.sum", 0)) / 1e9
    print(f"{i:>4} {names[i][0]:34s} {names[i][1]:>14s} {t:9.1f} us {gb:7.2f} GB {gb / t * 1e3 if t else 0:7.0f} GB/s "
          f"dmma {x.get('sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active', 0):5.1f}")
print(f"total {tot / 1e3:.2f} ms over {len(d)} launches")
if len(sys.argv) > 2 and sys.argv[2] == "--by-kernel":
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for i in d:
        a = agg[names[i][0]]
        a[0] += 1
        a[1] += d[i].get("gpu__time_duration.sum", 0) / 1e6
        a[2] += (d[i].get("dram__bytes_read.sum", 0) + d[i].get("dram__bytes_write.sum", 0)) / 1e9
    for k, (n, ms, gb) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{k:34s} n={n:3d} {ms:8.2f} ms {gb:7.1f} GB")
