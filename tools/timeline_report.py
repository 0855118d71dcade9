"""Summarise a K1 timeline CSV (profiling build: UM_GEMM_STALLS=1 UM_GEMM_TIMELINE=<csv>).

Per launch: span, tensor-side utilisation (sum of tile spans over pairs x
span), when the pulls land (10/50/90/100 % of chunks), and how long the pairs
sit before their first tile and after their last one."""
import csv
import sys
from collections import defaultdict

path = sys.argv[1]
only = set(int(x) for x in sys.argv[2].split(",")) if len(sys.argv) > 2 else None
tiles = defaultdict(list)
chunks = defaultdict(list)
with open(path) as f:
    for r in csv.DictReader(f):
        L = int(r["launch"])
        if only is not None and L not in only:
            continue
        if r["kind"] == "tile":
            tiles[L].append((int(r["pair"]), int(r["start_ns"]), int(r["end_ns"])))
        else:
            chunks[L].append(int(r["start_ns"]))
for L in sorted(set(tiles) | set(chunks)):
    ts = tiles[L]
    span = max([e for _, _, e in ts] + chunks[L] + [0])
    pairs = sorted({p for p, _, _ in ts})
    busy = sum(e - s for _, s, e in ts if e)
    util = busy / (len(pairs) * span) if pairs and span else 0.0
    first = sorted(min(s for p2, s, _ in ts if p2 == p) for p in pairs)
    last = sorted(max(e for p2, _, e in ts if p2 == p) for p in pairs)
    ch = sorted(chunks[L])

    def q(v, f):
        return v[min(len(v) - 1, int(f * (len(v) - 1)))] / 1e3 if v else 0.0

    print(f"launch {L}: span {span / 1e3:.1f} us, {len(ts)} tiles on {len(pairs)} pairs, MMA-side busy {util:.0%}; "
          f"first tile start median {q(first, .5):.1f} us (max {q(first, 1):.1f}); last tile end min {q(last, 0):.1f} us; "
          f"chunks {len(ch)} landed 10/50/90/100 % at {q(ch, .1):.1f}/{q(ch, .5):.1f}/{q(ch, .9):.1f}/{q(ch, 1):.1f} us")
