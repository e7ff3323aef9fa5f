# round 2 session 3: LL-size audit after the LL kernel went back to 40 registers -- every BASELINE schedule at 1-64 KiB, default vs channel / group grid, 2 repeats
make -s -j8 all > /dev/null
for rep in 1 2; do
timeout 1500 python tools/tune.py '{"scheds":["ag777","ag111","ring","ar822","ar56","ar_ring","a2a"],"sizes":[1024,8192,65536,262144],"knobs":[{},{"kb":1},{"kb":2},{"kb":4},{"kb":8},{"kb":16},{"kc":1,"kb":1},{"kc":8,"kb":1},{"kc":8,"kb":2},{"kc":56,"kb":1},{"kc":56,"kb":2}]}' >> gpurun_out/s3_ll_audit.jsonl 2>&1
done
python - <<'PY'
import json, collections
rows = [json.loads(l) for l in open("gpurun_out/s3_ll_audit.jsonl") if l.startswith("{") and '"us"' in l]
d = collections.defaultdict(list)
for r in rows: d[(r["sched"], r["bytes"], json.dumps(r["knobs"], sort_keys=True))].append((r["us"], r["kc"], r["kb"], r["proto"]))
base = {(s, b): min(v) for (s, b, k), v in d.items() if k == "{}"}
for (s, b), v in sorted(base.items()): print("BASE", s, b, v)
for (s, b, k), v in sorted(d.items()):
    if k == "{}" or (s, b) not in base: continue
    g = min(v)[0] / base[(s, b)][0]
    if g < 0.95: print(f"{s:8s} {b:>8d} {k:30s} {min(v)} vs {base[(s,b)]}  {100*(g-1):+.1f}%")
PY
