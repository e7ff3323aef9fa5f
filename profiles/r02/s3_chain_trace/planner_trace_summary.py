import json, collections, sys
import numpy as np
d=json.load(open(sys.argv[1])); ctas=d['ctas']
res=collections.defaultdict(list)
for key,v in ctas.items():
    ev=collections.defaultdict(dict)
    for t,meta in v:
        e=meta&0xff; op=(meta>>8)&0xffffff; tile=(meta>>32)
        if e==10: ev[(op,tile&0x7fffffff)]['have']=tile>>31
        if e in (1,8,9,10,11,7): ev[(op,tile&0x7fffffff)].setdefault(e,t)
    for k,e in ev.items():
        if 10 in e and 11 in e:
            res['planwait_have' if e['have'] else 'planwait_missing'].append((e[11]-e[10])/1e3)
        if 10 in e and 1 in e:
            res['planner_ahead_of_producer_flag'].append((e[1]-e[11])/1e3 if 11 in e else None)
for k,v in res.items():
    v=[x for x in v if x is not None]
    print(k, len(v), [round(float(np.quantile(v,q)),3) for q in (0.1,0.5,0.9)], 'sum/cta', round(sum(v)/len(ctas),1))
