import sys, numpy as np
sys.path.insert(0, ".")
import bench
import paper_2503_02356_b200 as cf
# measured fits (ms) from profiles/round1_step_breakdown (1-block C2 step)
F = (27.44, 7.0476e-3, 4.802e-7); B = (32.84, 1.7596e-2, 1.5998e-6); R = (0.0, 1.04457e-2, 4.767e-7)
def t(fit, T, pairs): return fit[0] + fit[1]*T + fit[2]*pairs
def units(N):
    lengths = np.concatenate([bench.block_lengths(b+1) for b in range(N)])
    plan = cf.Plan.build(lengths, bench.CHUNK, bench.K_RETAIN, np.arange(len(lengths)))
    ch, sg, _, _ = plan.export()
    us = {}
    groups = {}
    for c in ch:
        segs = sg[c["seg_offset"]:c["seg_offset"]+c["seg_count"]]
        if c["kind"] == 0:
            pairs = sum(float(s["length"])*(s["length"]+1)/2 for s in segs)
            us[("s", int(c["chunk_id"]))] = [(int(c["total_tokens"]), pairs, False)]
        else:
            s = segs[0]
            pairs = float(s["length"])*s["start_token"] + float(s["length"])*(s["length"]+1)/2
            groups.setdefault(int(s["sequence_id"]), []).append((int(c["total_tokens"]), pairs))
    for g, mem in groups.items():
        n = len(mem)
        us[("g", g)] = [(T, p, n > bench.K_RETAIN and i < n-bench.K_RETAIN) for i, (T, p) in enumerate(mem)]
    return list(us.values())
def measured(u):
    return sum(t(F,T,p)+t(B,T,p)+(t(R,T,p) if rc else 0) for T,p,rc in u)
def model(u, gamma, beta, rfrac):
    return sum((gamma + T + beta*p)*(1+(rfrac if rc else 0)) for T,p,rc in u)
def lpt(costs, N):
    order = sorted(range(len(costs)), key=lambda i: -costs[i])
    load = [0.0]*N; out=[[] for _ in range(N)]
    for i in order:
        b = min(range(N), key=lambda r: load[r]); load[b]+=costs[i]; out[b].append(i)
    return out
for N in [1,2,4,8]:
    us = units(N)
    meas = [measured(u) for u in us]
    for name, w in [("old", (0, 4.4e-5, 1/3)), ("new", (2440, 8.4e-5, 0.29))]:
        parts = lpt([model(u,*w) for u in us], N)
        rt = [sum(meas[i] for i in p) for p in parts]
        print(N, name, "max/mean %.4f" % (max(rt)/np.mean(rt)), "max ms %.0f" % max(rt), "ideal %.0f" % (sum(meas)/N))
