"""Spread of per-CTA trace end times in a NUFI_STAMPS file (python tools/cta_end.py /tmp/stamps_sl1.txt).
Entries are (globaltimer << 8 | smid) truncated to 64 bits: times are compared modulo 2^56."""
import collections
import sys

import numpy as np

for l in open(sys.argv[1]):
    if not l.startswith("# cta trace end"):
        continue
    step = l.split(",")[1].split(":")[0]
    raw = [int(x) for x in l.split(":")[1].split()]
    t = np.array([(x >> 8) for x in raw], dtype=np.float64)
    sm = np.array([x & 0xFF for x in raw])
    t -= t.min()
    print(step, "n_ctas", len(t), "end spread us: p10 %.1f p50 %.1f p90 %.1f max %.1f" % tuple(
        np.percentile(t, q) / 1e3 for q in (10, 50, 90, 100)))
    order = np.argsort(t)[-6:]
    print("  latest CTAs (idx, sm, us):", [(int(i), int(sm[i]), round(t[i] / 1e3, 1)) for i in order])
    d = collections.defaultdict(list)
    for i in range(len(t)):
        d[int(sm[i])].append(i)
    print("  CTAs per SM:", dict(collections.Counter(len(x) for x in d.values())))
    # CTA index parity / position
    print("  mean end by CTA idx decile (us):", [round(float(np.mean(t[k * len(t) // 10:(k + 1) * len(t) // 10])) / 1e3, 1) for k in range(10)])
