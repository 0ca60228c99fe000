"""Summarise a pair-gather event timeline (LUTGPU_OH_TL=<file>) as median latencies."""
import collections
import csv
import statistics as st
import sys

ev = collections.defaultdict(dict)
for r in csv.DictReader(open(sys.argv[1])):
    ev[(int(r["cta"]), int(r["event"]))][int(r["idx"])] = int(r["ns"])


def d(c1, e1, c2, e2, rng, off=0):
    xs = [ev[(c2, e2)][g + off] - ev[(c1, e1)][g] for g in rng if g in ev[(c1, e1)] and g + off in ev[(c2, e2)]]
    return st.median(xs) if xs else float("nan")


R = range(20, 180)
print("gen L: built->emptyok %.0f emptyok->arrive %.0f | P: arrive->sigfwd %.0f sigfwd->M.afull %.0f | L.arrive->M.afull %.0f"
      % (d(0, 0, 0, 1, R), d(0, 1, 0, 2, R), d(1, 2, 1, 3, R), d(1, 3, 0, 4, R), d(0, 2, 0, 4, R)))
print("M: afull->issued %.0f ; issued(g)->L.emptyok(g+3) %.0f P %.0f" % (d(0, 4, 0, 5, R), d(0, 5, 0, 1, R, 3), d(0, 5, 1, 1, R, 3)))
xs = sorted(ev[(0, 4)].items())
per = [xs[i + 1][1] - xs[i][1] for i in range(20, len(xs) - 1)]
print("MMA stage period median %.0f mean %.0f ns" % (st.median(per), sum(per) / len(per)))
seq = [(7, "accfull"), (11, "wait_read0"), (12, "ld0"), (13, "math0"), (14, "ld1"), (8, "rel"), (15, "math1"), (9, "loopend"),
       (16, "fence"), (10, "stores")]
U = range(5, 150)
for c in (0, 1):
    parts = []
    for (e1, n1), (e2, n2) in zip(seq, seq[1:]):
        parts.append("%s->%s %.0f" % (n1, n2, d(c, e1, c, e2, U)))
    ys = sorted(ev[(c, 7)].items())
    per = [ys[i + 1][1] - ys[i][1] for i in range(5, len(ys) - 1)]
    print("epi cta%d: " % c + ", ".join(parts) + " | unit period %.0f" % st.median(per))
print("M.accempty_ok(u) - L.epi.rel(u-2) %.0f" % d(0, 8, 0, 6, range(5, 150), 2))
# per-unit MMA issuer breakdown: wait for acc_empty (epilogue-bound) vs the 4 a_full waits (generator-bound)
nst = 4
wa, wf, busy = [], [], []
for u in range(6, 150):
    try:
        prev_issue = ev[(0, 5)][nst * u - 1]
        ok = ev[(0, 6)][u]
        wa.append(ok - prev_issue)
        t = ok
        for g in range(nst * u, nst * u + nst):
            wf.append(ev[(0, 4)][g] - t)
            busy.append(ev[(0, 5)][g] - ev[(0, 4)][g])
            t = ev[(0, 5)][g]
    except KeyError:
        pass
if wa:
    print("MMA per unit: wait acc_empty %.0f ns, wait a_full %.0f ns (4 stages), issue %.0f ns (4 stages)"
          % (st.mean(wa), 4 * st.mean(wf), 4 * st.mean(busy)))
# epilogue release skew: peer vs leader
print("epi release skew peer-leader %.0f ns" % d(0, 8, 1, 8, range(5, 150)))
