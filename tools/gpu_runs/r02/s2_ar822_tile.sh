# round 2 session 2: one-shot allreduce (pull, fan-in 8) tile size at 2-48 MiB per rank, 3 repeats
for rep in 1 2 3; do
timeout 900 python tools/tune.py '{"scheds":["ar822"],"sizes":[2097152,4194304,8388608,12582912,16777216,33554432,50331648],"knobs":[{},{"tile":16384},{"tile":32768}]}' >> gpurun_out/s2_ar822_tile.jsonl 2>&1
done
python - <<'PY'
import json, collections
d = collections.defaultdict(list)
for l in open("gpurun_out/s2_ar822_tile.jsonl"):
    if l.startswith("{") and '"us"' in l:
        r = json.loads(l); d[(r["bytes"], json.dumps(r["knobs"]), r["tile"], r["grid"])].append(r["us"])
for k in sorted(d): print(k, sorted(d[k]))
PY
