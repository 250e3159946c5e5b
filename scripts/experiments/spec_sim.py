"""Simulate segment-speculative greedy CTC: from a cold start (root, last=argmax[f0-1])
at frame f0, how many frames until the trajectory's entry (state, last) equals the truth."""
import sys, numpy as np
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import gen_inputs as gi
from oracle import oracle as orc
phrases, V = gi.corpus("p20k_v1024")
tab = orc.build_table(phrases, V)
cache = {}
def row(s):
    if s not in cache:
        sc, nx = orc.score_batch(tab, np.array([s], np.int32)); cache[s] = (sc[0].astype(np.float64), nx[0])
    return cache[s]
def step(lp, a, t, state, last, lam=1.0, blank=0):
    if a[t] == blank or a[t] == last: return state, a[t]
    sc, nx = row(state)
    comb = lp[t].astype(np.float64) + lam * sc
    comb[blank] = -np.inf
    if last >= 0: comb[last] = -np.inf
    best = comb.max(); cand = np.flatnonzero(comb == best)
    if cand.size > 1: r = lp[t][cand]; cand = cand[r == r.max()]
    ch = int(cand[0]); return int(nx[ch]), ch
rng = np.random.default_rng(5)
regime = sys.argv[1] if len(sys.argv) > 1 else "dense"
T = 200; delays = []; changed = 0; emits = 0
for u in range(int(sys.argv[2]) if len(sys.argv) > 2 else 8):
    lg = rng.normal(0, 2.0, size=(T, V))
    if regime == "blank3": lg[np.arange(T) % 4 != 0, 0] += 10
    lp = gi.log_softmax(lg).astype(np.float32); a = lp.argmax(1)
    ent = []; st, last = 0, -1
    for t in range(T):
        ent.append((st, last)); ns, nl = step(lp, a, t, st, last)
        if not (a[t] == 0 or a[t] == last): emits += 1; changed += nl != a[t]
        st, last = ns, nl
    for f0 in range(8, T - 40, 7):
        st, last = 0, int(a[f0 - 1])
        for t in range(f0, T):
            if (st, last) == ent[t]: delays.append(t - f0); break
            st, last = step(lp, a, t, st, last)
        else: delays.append(999)
d = np.array(delays)
print(regime, "emitting", emits, "boost-changed", changed, "sync delay: mean", d.mean(), "pcts", np.percentile(d, [50, 90, 99, 100]))
print("hist", np.bincount(np.minimum(d, 40)))
