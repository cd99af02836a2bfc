"""Compare two root_profile logs per level class (diagnostics).
  python tools/ab_levels.py A.log B.log"""
import json
import sys


def load(f):
    return {d["root"]: d for d in map(json.loads, open(f)) if "root" in d}


A, B = load(sys.argv[1]), load(sys.argv[2])
agg = {}
for r in A:
    a, b = A[r], B.get(r)
    if not b or a["trace"] != b["trace"]:
        continue
    for i, (d, c) in enumerate(zip(a["trace"], a["claims"])):
        if i >= len(a["level_us"]) or i >= len(b["level_us"]):
            continue
        prev = a["trace"][i - 1] if i else "-"
        key = (prev + d, "small" if c < 1e4 else ("mid" if c < 1e6 else "big"))
        x = agg.setdefault(key, [0, 0, 0])
        x[0] += a["level_us"][i]
        x[1] += b["level_us"][i]
        x[2] += 1
    for k, fa, fb in (("init", a["init_us"], b["init_us"]),
                      ("rest", a["kernel_us"] - sum(a["level_us"]), b["kernel_us"] - sum(b["level_us"])),
                      ("total", a["kernel_us"], b["kernel_us"])):
        x = agg.setdefault((k,), [0, 0, 0])
        x[0] += fa
        x[1] += fb
        x[2] += 1
for k, v in sorted(agg.items(), key=str):
    print(f"  {str(k):24s} A {v[0] / v[2]:8.1f}  B {v[1] / v[2]:8.1f}  n {v[2]}")
