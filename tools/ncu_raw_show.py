"""Print the metrics of an `ncu --page raw --csv` export: python tools/ncu_raw_show.py FILE..."""
import csv, sys
for f in sys.argv[1:]:
    rows = list(csv.reader(open(f)))
    h = [i for i, r in enumerate(rows) if r and r[0] == "ID"]
    if not h:
        print(f, "no data"); continue
    hdr, val = rows[h[0]], rows[h[0] + 2]
    print(f)
    for k, v in zip(hdr, val):
        if k.startswith(("gpu__", "smsp", "sm__", "l1tex", "launch__", "lts__", "dram__")):
            print("  %-80s %s" % (k, v))
