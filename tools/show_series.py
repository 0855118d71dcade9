"""Summarise tagged k1_series.py output lines: tag impl kernel-MHz median best TF/GHz."""
import json
import sys

for path in sys.argv[1:]:
    for line in open(path):
        tag, _, rest = line.partition(" ")
        if rest.startswith("{"):
            d = json.loads(rest)
            mhz = d.get("kernel_mhz") or 0
            print(f"{tag:28s} {d['impl']:3s} kmhz {mhz:5d} med {d['median']:6.0f} best {d['best']:6.0f} "
                  f"TF/GHz {d['median'] / mhz * 1000 if mhz else 0:5.0f}")
        else:
            print(line.rstrip()[:300])
