"""Replays the forward's measured per-task cycles (FWDTASK records of a
-DSKEI_FWD_STATS -DSKEI_FWD_STATS_TASKS build: tools/fwd_stats.py with STATS_RAW, or the CSV
kept in profiles/r2_fwd_task_cycles_s5.csv) through alternative static task-to-warp deals
(snake, snake with reversed rounds, least-loaded warp; by estimated cost, by block count, by
the measured cycles themselves) and prints each deal's max / mean of the warps' task cycles.

    python tools/fwd_task_deal.py profiles/r2_fwd_task_cycles_s5.csv
"""
import re, collections, numpy as np, sys
pat=re.compile(r'cta (\d+) warp (\d+) slot (\d+) ab1e4 (\d+) c0 (\d+) cost (\d+) blocks (\d+) cycles (\d+) cls (\d+)')
units=[]  # list of dict (warp,slot)->row
cur={}
for l in open(sys.argv[1]):
    m=pat.search(l)
    if m:
        v=list(map(int,m.groups()))
    elif re.match(r'^\d+(,\d+){8}$', l.strip()):
        v=list(map(int,l.strip().split(',')))
    else:
        continue
    d=cur.setdefault(v[0],{})
    if (v[1],v[2]) in d:
        units.append(d); d={}; cur[v[0]]=d
    d[(v[1],v[2])]=v
units+= [d for d in cur.values() if d]
units=[u for u in units if len(u)>=40]
print(len(units),"units; tasks per unit:",collections.Counter(len(u) for u in units))
def deal_eval(assign, cyc):  # assign: list of warp per task
    L=np.zeros(16)
    for w,c in zip(assign,cyc): L[w]+=c
    return L.max()/L.mean(), L.max()
res=collections.defaultdict(list)
for u in units:
    rows=np.array(list(u.values()))
    warp,slot,ab,c0,cost,blocks,cyc=rows[:,1],rows[:,2],rows[:,3],rows[:,4],rows[:,5],rows[:,6],rows[:,7]
    res['actual'].append(deal_eval(warp,cyc)[0])
    def by_rank(key, pattern):
        order=np.lexsort((np.arange(len(key)),-key))
        asg=np.zeros(len(key),int)
        for r,i in enumerate(order):
            rd,wi=divmod(r,16)
            asg[i]= 15-wi if pattern[rd] else wi
        return asg
    res['snake FRFR est'].append(deal_eval(by_rank(cost,[0,1,0,1]),cyc)[0])
    res['snake FRRF est'].append(deal_eval(by_rank(cost,[0,1,1,0]),cyc)[0])
    res['snake FRFR blocks'].append(deal_eval(by_rank(blocks,[0,1,0,1]),cyc)[0])
    res['snake FRRF blocks'].append(deal_eval(by_rank(blocks,[0,1,1,0]),cyc)[0])
    def lpt(key):
        order=np.lexsort((np.arange(len(key)),-key)); L=np.zeros(16); asg=np.zeros(len(key),int)
        for i in order:
            w=int(np.argmin(L)); L[w]+=key[i]; asg[i]=w
        return asg
    res['LPT est'].append(deal_eval(lpt(cost),cyc)[0])
    res['LPT blocks'].append(deal_eval(lpt(blocks),cyc)[0])
    res['LPT act'].append(deal_eval(lpt(cyc),cyc)[0])
    # model: cycles ~ blocks*(a + b*wtnorm)
    for bw in (0.0,0.1,0.2,0.3):
        wtn=cost/np.maximum(blocks,1)/16.0
        key=blocks*(1+bw*(wtn-1))
        res[f'LPT blocks*(1+{bw}(wt-1))'].append(deal_eval(lpt(key),cyc)[0])
        res[f'snakeFRFR blocks*(1+{bw}(wt-1))'].append(deal_eval(by_rank(key,[0,1,0,1]),cyc)[0])
for k,v in res.items(): print(f"{k:40s} max/mean {np.mean(v):.3f}")
