# round 2 session 2: (7,7,7) allgather, chunk-group split (default kc=2) vs kc=1, alternating, 3 repeats
for rep in 1 2 3; do
timeout 900 python tools/tune.py '{"scheds":["ag777","ring"],"sizes":[67108864,134217728,268435456,536870912],"knobs":[{},{"kc":1,"kb":37}]}' >> gpurun_out/s2_ag_split_ab.jsonl 2>&1
done
python - <<'PY'
import json, collections
d = collections.defaultdict(list)
for l in open("gpurun_out/s2_ag_split_ab.jsonl"):
    if l.startswith("{"):
        r = json.loads(l); d[(r["sched"], r["bytes"], r["kc"])].append(r["us"])
for k in sorted(d): print(k, sorted(d[k]))
PY
