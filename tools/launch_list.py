"""ncu launch-list CSV (--metrics gpu__time_duration.sum --csv --log-file) of
tools/prof_gen.py -> the kernels of the last generation, one line each.
usage: launch_list.py launches.csv "title" > launches.txt"""
import csv, sys
rows = []
with open(sys.argv[1]) as fh:
    lines = [l for l in fh if l.startswith('"')]
rd = csv.DictReader(lines)
for r in rd:
    if r.get("Metric Name") != "gpu__time_duration.sum":
        continue
    v = float(r["Metric Value"].replace(",", ""))
    unit = r.get("Metric Unit", "ns")
    us = v / 1e3 if unit in ("ns", "nsecond") else (v if unit in ("us", "usecond") else v * 1e3)
    rows.append((r["Kernel Name"], us))
# the last generation starts at the last k_sample / k_keys_from_coords launch
start = max((i for i, (k, _) in enumerate(rows) if "k_sample(" in k or k.startswith("hrg::k_sample")
             or "k_shard_keys" in k), default=0)
rows = rows[start:]
print("# " + (sys.argv[2] if len(sys.argv) > 2 else ""))
for k, us in rows:
    print(f"{us:9.1f} us  {k[:100]}")
print(f"total {sum(us for _, us in rows):.1f} us")
