"""Reconstructs a DAG for Fig. 9 (P:L204 caption, P:L233 text "the DAG's makespan increases from
11 to 14 units"; per-call durations are not given, the DAG is DERIVED by exhaustive
search).  Criteria: one program, one root, BS = 2 slots, non-preemptive work-conserving list
scheduling; critical path 11; the best list order reaches 11 (critical-path-first), the worst
reaches 14, and FCFS in call-index order is the worst.  Output went to tests/golden/fig9.json
(the 5-call hit).  Independent of oracle/ and of the CUDA path."""
import itertools, random
def listsched(dur, par, order, m=2):
    n=len(dur); done=[None]*n; t=0; running={}  # call->end
    started=set(); rank={c:i for i,c in enumerate(order)}
    while len([c for c in range(n) if done[c] is not None])<n:
        # free slots
        ready=[c for c in range(n) if c not in started and all(done[p] is not None and done[p]<=t for p in par[c])]
        ready.sort(key=lambda c: rank[c])
        while len(running)<m and ready:
            c=ready.pop(0); started.add(c); running[c]=t+dur[c]
        t2=min(running.values()); t=t2
        for c in [c for c,e in running.items() if e==t]:
            done[c]=t; del running[c]
    return max(done)
def cp(dur,par):
    f=[0]*len(dur)
    for c in range(len(dur)):
        f[c]=max([f[p] for p in par[c]],default=0)+dur[c]
    return max(f)
random.seed(1)
best=None
for trial in range(200000):
    n=random.randint(4,7)
    dur=[random.randint(1,6) for _ in range(n)]
    par=[sorted(random.sample(range(c),random.randint(0,min(2,c)))) if c else [] for c in range(n)]
    if cp(dur,par)!=11 or sum(1 for p in par if not p)!=1: continue
    ms=[listsched(dur,par,o) for o in itertools.permutations(range(n))]
    if min(ms)==11 and max(ms)==14 and listsched(dur,par,list(range(n)))==14:
        print(n,dur,par,sum(dur)); 
        if best is None or sum(dur)<best[0]: best=(sum(dur),n,dur,par)
        if n<=5: break
print(best)
