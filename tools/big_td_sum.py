"""Sum of the large top-down level times (> 2e7 frontier edges) in root_profile
logs (diagnostics: A/B of the top-down claim path at scale 26).
  python tools/big_td_sum.py A.log B.log ..."""
import json
import sys


def load(f):
    return [json.loads(line) for line in open(f) if line.startswith('{"root"')]


for f in sys.argv[1:]:
    tot, n = 0.0, 0
    for x in load(f):
        for L, (t, e) in enumerate(zip(x["trace"], x["td_edges"])):
            if t == "t" and e and e > 2e7 and L < len(x["level_us"]):
                tot += x["level_us"][L]
                n += 1
    print(f, "big TD levels", n, "sum us %.0f" % tot)
