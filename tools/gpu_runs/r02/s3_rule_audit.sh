# round 2 session 3: stale-rule audit with the final kernel -- every BASELINE schedule x size against single-knob deviations, 2 repeats
make -s -j8 all > /dev/null
for rep in 1 2; do
timeout 1500 python tools/tune.py '{"scheds":["ag777","ag111","ring","ar822","ar56","ar_ring","a2a"],"sizes":[262144,1048576,4194304,16777216,67108864,268435456],"knobs":[{},{"env":{"SCCL_WINDOW":"0"}},{"env":{"SCCL_WINDOW":"32768"}},{"env":{"SCCL_L2HINT":"1"}},{"env":{"SCCL_L2HINT":"0"}},{"env":{"SCCL_DISCARD":"1"}},{"env":{"SCCL_DISCARD":"0"}},{"tile":16384},{"tile":65536,"budget":196608},{"env":{"SCCL_SELFPUB":"1"}},{"env":{"SCCL_SELFPUB":"0"}},{"protocol":"simple"},{"protocol":"ll"}]}' >> gpurun_out/s3_rule_audit.jsonl 2>&1
done
python - <<'PY'
import json, collections
rows = [json.loads(l) for l in open("gpurun_out/s3_rule_audit.jsonl") if l.startswith("{") and '"us"' in l]
d = collections.defaultdict(list)
for r in rows: d[(r["sched"], r["bytes"], json.dumps(r["knobs"], sort_keys=True))].append(r["us"])
base = {(s, b): min(v) for (s, b, k), v in d.items() if k == "{}"}
for (s, b, k), v in sorted(d.items()):
    if k == "{}" or (s, b) not in base: continue
    g = min(v) / base[(s, b)]
    if g < 0.97: print(f"{s:8s} {b:>10d} {k:45s} {min(v):9.2f} vs {base[(s,b)]:9.2f}  {100*(g-1):+.1f}%")
PY
