# round 2 session 2: GPU suite after the tile / chunk-group policy changes, ar822 hint check
set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/s2v_smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q -rs > gpurun_out/s2v_pytest_gpu.log 2>&1
for rep in 1 2 3; do
timeout 600 python tools/tune.py '{"scheds":["ar822"],"sizes":[67108864,134217728,268435456],"knobs":[{},{"env":{"SCCL_L2HINT":"0"}}]}' >> gpurun_out/s2v_ar822_hint.jsonl 2>&1
done
tail -3 gpurun_out/s2v_pytest_gpu.log
python - <<'PY'
import json, collections
d = collections.defaultdict(list)
for l in open("gpurun_out/s2v_ar822_hint.jsonl"):
    if l.startswith("{") and '"us"' in l:
        r = json.loads(l); d[(r["bytes"], json.dumps(r["knobs"]))].append(r["us"])
for k in sorted(d): print(k, sorted(d[k]))
PY
