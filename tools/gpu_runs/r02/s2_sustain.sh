# round 2 session 2: burst vs sustained per-launch time of the bench workload
python tools/probes/sustain_probe.py $((128<<20)) > gpurun_out/s2_sustain.jsonl 2>&1
python tools/probes/sustain_probe.py $((128<<20)) 1 37 >> gpurun_out/s2_sustain.jsonl 2>&1
cat gpurun_out/s2_sustain.jsonl
