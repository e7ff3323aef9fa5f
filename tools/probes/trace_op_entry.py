#!/usr/bin/env python3
"""Producer cost at op boundaries from a raw trace dump (trace_chain.py with
TRACE_DUMP=<file>): per op's first tile, setup = TR_ENTRY - TR_ISSUED of the
previous tile (loop, descriptors, addresses) and flagwait = TR_FLAG -
TR_ENTRY (receipt counter read), split by whether the tile has a receipt
input.  usage: python tools/probes/trace_op_entry.py dump.json"""
import json, statistics, collections, sys
import numpy as np
d=json.load(open(sys.argv[1]))
prog=d['program']; ctas=d['ctas']; P=8
ranks=prog['ranks']
off=[0]
for r in range(P): off.append(off[-1]+len(ranks[r]['ops']))
res=collections.defaultdict(list)
for key,v in ctas.items():
    ev=collections.defaultdict(dict); entry={}
    for t,meta in v:
        e=meta&0xff; op=(meta>>8)&0xffffff; tile=(meta>>32)
        if e==9: entry[op]=t; continue
        if e in (0,5,6): continue
        ev[(op,tile&0x7fffffff)].setdefault(e,t)
        if e==1: ev[(op,tile&0x7fffffff)]['w']=tile>>31
    keys=sorted([k for k in ev if 1 in ev[k] and 8 in ev[k]], key=lambda k: ev[k][1])
    prev=None
    for k in keys:
        e=ev[k]
        if k[1]==0 and k[0] in entry and prev is not None:
            tag='rcpt' if e['w'] else 'none'
            res['setup_'+tag].append((entry[k[0]]-prev)/1e3)
            res['flagwait_'+tag].append((e[1]-entry[k[0]])/1e3)
        prev=e[8]
for k,v in sorted(res.items()): print(k, len(v), [round(float(np.quantile(v,q)),3) for q in (0.1,0.5,0.9)], 'sum/cta', round(sum(v)/len(ctas),1))
