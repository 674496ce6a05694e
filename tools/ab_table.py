"""Summarise tools/ab_lib.py output (dev tool): mean GB/s per library per workload,
relative to the first library.  python tools/ab_table.py AB.txt"""
import collections
import re
import sys

d = collections.OrderedDict()
order = []
for line in open(sys.argv[1]):
    m = re.search(r"(\S+?)(?:@(\S+))?: op=(\d) dim=(\d) (?:cfg|regime)=(\S+) (f\d\d) ([\d.]+) ms/launch, ([\d.]+) GB/s", line)
    if not m:
        continue
    lib = m.group(1).split("/")[-1] + ("@" + m.group(2) if m.group(2) else "")
    key = "op%s dim%s %s %s" % m.group(3, 4, 5, 6)
    d.setdefault(key, collections.OrderedDict()).setdefault(lib, []).append(float(m.group(8)))
    if lib not in order:
        order.append(lib)
print("workload".ljust(22) + "".join(l[:16].rjust(17) for l in order))
for key, v in d.items():
    base = sum(v[order[0]]) / len(v[order[0]]) if order[0] in v else None
    cells = []
    for lib in order:
        if lib not in v:
            cells.append("-".rjust(17))
            continue
        g = sum(v[lib]) / len(v[lib])
        cells.append(("%.0f (%+.1f%%)" % (g, 100 * (g / base - 1)) if base else "%.0f" % g).rjust(17))
    print(key.ljust(22) + "".join(cells))
