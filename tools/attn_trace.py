"""Summarise a CF_ATTN_TRACE=1 timeline of the persistent dQ kernel (CTA 0):
where the MMA issuer and softmax warp 0 spend their cycles.
Usage: CF_LIB=build_ab/lib_trace.so CF_TRACE_OUT=t.txt python tools/attn_short_bench.py 14
       python tools/attn_trace.py t.txt"""
import collections
import sys

launches, cur = [], None
for line in open(sys.argv[1]):
    if line.startswith("#"):
        cur = []
        launches.append(cur)
        continue
    r, t, ev, j = (int(x) for x in line.split())
    cur.append((r, t, ev, j))
ev = launches[-1]
mma = [(t, e, j) for r, t, e, j in ev if r == 0]
smx = [(t, e, j) for r, t, e, j in ev if r == 1]
t0 = min(t for _, t, _, _ in ev)
t1 = max(t for _, t, _, _ in ev)
print(f"launches traced {len(launches)}; last: CTA 0 span {t1 - t0} cycles, mma events {len(mma)}, softmax events {len(smx)}")

# MMA issuer: time between consecutive events, attributed to the wait that ends at the later event
names_m = {1: "issue_s start", 2: "K/V ready (wait K/V)", 3: "S buffer free (wait s_free)", 4: "item start",
           5: "Q/dO staged (wait q_full)", 6: "dS ready (wait ds_full)", 7: "dQ buffer free (wait dq_free)"}
names_s = {1: "loop top", 2: "S/dP done (wait s_full)", 3: "softmax math + tmem ld", 4: "dS slot free (wait ds_free)",
           5: "item MMAs done (wait dq_done)", 6: "next item staged (stage)", 7: "dQ read out + stored"}
for title, seq, names in (("MMA issuer", mma, names_m), ("softmax warp 0", smx, names_s)):
    acc = collections.Counter()
    for (ta, ea, ja), (tb, eb, jb) in zip(seq, seq[1:]):
        acc[eb] += tb - ta
    tot = sum(acc.values())
    print(f"== {title}: {tot} cycles between first and last event")
    for e, c in sorted(acc.items(), key=lambda kv: -kv[1]):
        print(f"   {names[e]:34s} {c:9d}  {100 * c / max(tot, 1):5.1f}%")
items = sum(1 for _, e, _ in mma if e == 4)
subs = sum(1 for _, e, _ in mma if e == 7)
print(f"items {items}, sub-tiles {subs}, cycles per sub-tile {(t1 - t0) / max(subs, 1):.0f}")
