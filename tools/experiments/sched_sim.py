"""Fluid model of the C2 forward grid on 592 SM sub-partitions (DESIGN.md §7
"Where C2 loses"): jobs of 20 chunks, per-sub-partition throughput F[k]
chunks/us with k forward warps (measured: lone 4.2 us/chunk, two warps
7.0 us/chunk each), traceback 15 us, and a job move costing h us.  Compares
the static placement with a work queue whose jobs move at segment boundaries
(policy "alone": a job keeps running if it is alone on its sub-partition)."""
import random, numpy as np
from collections import deque
F = [0, 0.238, 0.286, 0.300, 0.31]
def run(njobs=1026, nchunk=20, Q=5, slots=2, nsm=592, h=1.0, tb=14.7, dt=0.05, cont="alone", prio="level", var=0.0, seed=1):
    rnd = random.Random(seed)
    nw = nsm*slots
    sm = [i % nsm for i in range(nw)]
    spd = [1.0 + var*(rnd.random()-0.5) for _ in range(nsm)]
    state = ['wait']*nw; rem=[0.0]*nw; job=[None]*nw; pos=[0]*nw; segend=[0]*nw; tu=[0.0]*nw
    waiting = deque(range(nw))
    nseg=(nchunk+Q-1)//Q
    levels=[deque() for _ in range(nchunk+1)]
    for j in range(njobs): levels[0].append(j)
    t=0.0; done=0; fe=[]; hand=0
    def pop():
        for c in range(nchunk+1):
            if levels[c]: return levels[c].popleft(), c
        return None
    def minlevel():
        for c in range(nchunk+1):
            if levels[c]: return c
        return 99
    def begin(w, j, c, load):
        job[w]=j; pos[w]=c; segend[w]=min((c//Q+1)*Q, nchunk); rem[w]=segend[w]-c
        state[w]='load' if load else 'fwd'; tu[w]=t+h
    def dispatch():
        while waiting:
            u = pop()
            if u is None: break
            w = waiting.popleft(); begin(w,u[0],u[1],True)
    dispatch()
    while done < njobs:
        cnt=[0]*nsm
        for w in range(nw):
            if state[w] in ('fwd','load'): cnt[sm[w]]+=1
        for w in range(nw):
            s=state[w]
            if s=='load' and t>=tu[w]: state[w]='fwd'
            elif s=='fwd':
                kk = cnt[sm[w]]
                rem[w]-=F[kk]/kk*spd[sm[w]]*dt
                if rem[w]<=0:
                    if segend[w]>=nchunk:
                        state[w]='tb'; tu[w]=t+tb; fe.append(t)
                    else:
                        keep = False
                        if cont=="alone": keep = cnt[sm[w]]<=1
                        elif cont=="alone_or_ahead": keep = cnt[sm[w]]<=1 or segend[w] < minlevel()
                        elif cont=="never": keep=False
                        elif cont=="always": keep=True
                        if keep: begin(w, job[w], segend[w], False)
                        else:
                            levels[segend[w]].append(job[w]); state[w]='wait'; waiting.append(w); cnt[sm[w]]-=1; hand+=1
            elif s=='tb' and t>=tu[w]:
                done+=1; state[w]='wait'; waiting.append(w)
        dispatch()
        t+=dt
    fe=np.array(fe)
    return round(t,1), hand, [round(np.percentile(fe,x),1) for x in (0,50,100)]
for var in ():
  for cont in ("always","alone","never","alone_or_ahead"):
    for Q in (5,4,2,1):
      print(var, cont, "Q",Q, run(Q=Q,cont=cont,var=var,h=1.0))
print("---- realistic F")
for h in (1.0, 2.0, 6.0):
  for cont in ("always","alone"):
    for Q in (4,2,1):
      print("h",h, cont, "Q",Q, run(Q=Q,cont=cont,var=0.0,h=h))
