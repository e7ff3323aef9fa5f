# round 2 session 2: simple-protocol chunk groups limited to the chunks a rank works on (new) vs HEAD, alternating, 2 repeats
G='{"scheds":["ag111","ar822"],"sizes":[16384,65536,262144,524288,1048576,4194304],"knobs":[{},{"protocol":"simple"}]}'
for rep in 1 2; do
  SCCL_LIB=build/ab/libsccl_exec_head.so timeout 600 python tools/tune.py "$G" | sed 's/^{/{"lib": "head", /' >> gpurun_out/s2_workchunks_ab.jsonl 2>&1
  timeout 600 python tools/tune.py "$G" | sed 's/^{/{"lib": "new", /' >> gpurun_out/s2_workchunks_ab.jsonl 2>&1
done
python - <<'PY'
import json, collections
d = collections.defaultdict(list)
for l in open("gpurun_out/s2_workchunks_ab.jsonl"):
    if l.startswith("{") and '"us"' in l:
        r = json.loads(l); d[(r["sched"], r["bytes"], json.dumps(r["knobs"]), r["lib"])].append((r["us"], r["kc"], r["kb"], r["proto"]))
keys = sorted({k[:3] for k in d})
for k in keys:
    h, n = min(d[k + ("head",)]), min(d[k + ("new",)])
    print(k, "head", h, "new", n, f"{100*(n[0]/h[0]-1):+.1f}%")
PY
