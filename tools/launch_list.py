"""Format an ncu --csv launch list (gpu__time_duration.sum [+ grid/block]) as
the per-launch table kept under profiles/.  usage: launch_list.py CSV [header...]"""
import csv
import re
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) >= 15 and r[0].isdigit()]
launches = {}
for r in rows:
    i = int(r[0])
    name = re.sub(r"^.*::", "", r[4].split("(")[0]) if "(" in r[4] else r[4]
    name = re.sub(r"\(.*", "", name)
    e = launches.setdefault(i, {"name": name, "grid": r[8], "block": r[7]})
    e[r[12]] = r[14]
for line in sys.argv[2:]:
    print("# " + line)
print(f"# {'id':>3}  {'kernel':28s} {'grid':>14s} {'block':>12s} {'ns':>10s}")
tot = 0
for i in sorted(launches):
    e = launches[i]
    ns = int(float(e.get("gpu__time_duration.sum", "0").replace(",", "")))
    tot += ns
    g = e["grid"].strip("()").split(",")[0]
    b = e["block"].strip("()").split(",")[0]
    print(f"  {i:3d}  {e['name'][:28]:28s} {g:>14s} {b:>12s} {ns:10d}")
print(f"# total {tot} ns over {len(launches)} launches")
