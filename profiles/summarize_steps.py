"""Launch-list summary of the decode steps only: the rows of an ncu
--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
--csv log from profiles/prof_decode.py, from the first la_step_build_kernel on
(the prefill before it is left out).  Per kernel: launches, mean duration,
share of the steps' serialised kernel time, DRAM bytes per launch.
    python profiles/summarize_steps.py gpurun_out/r02e_launches.csv"""
import collections
import csv
import io
import sys

txt = open(sys.argv[1]).read().splitlines()
start = next(i for i, l in enumerate(txt) if l.startswith('"ID"'))
rows = list(csv.DictReader(io.StringIO("\n".join(txt[start:]))))
launch = collections.OrderedDict()   # ID -> {name, metrics}
for r in rows:
    d = launch.setdefault(r["ID"], {"name": r["Kernel Name"]})
    d[r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
ids = list(launch)
first = next(i for i, k in enumerate(ids) if launch[k]["name"].startswith("la_step_build_kernel"))
agg = collections.OrderedDict()
for k in ids[first:]:
    d = launch[k]
    name = d["name"].split("(")[0].replace("void <unnamed>::", "").replace("<unnamed>::", "")
    a = agg.setdefault(name, [0, 0.0, 0.0])
    a[0] += 1
    a[1] += d.get("gpu__time_duration.sum", 0.0)
    a[2] += d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
tot = sum(a[1] for a in agg.values())
steps = sum(1 for k in ids[first:] if launch[k]["name"].startswith("la_step_build_kernel"))
print(f"# {steps} decode steps, {len(ids) - first} launches, serialised kernel time {tot / 1e3 / steps:.1f} us per step")
print(f"# {'kernel':34s} {'n':>5s} {'mean us':>9s} {'share':>7s} {'DRAM MB/launch':>15s}")
for name, (n, t, b) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"  {name:34s} {n:5d} {t / n / 1e3:9.2f} {t / tot * 100:6.1f}% {b / n / 1e6:15.2f}")
