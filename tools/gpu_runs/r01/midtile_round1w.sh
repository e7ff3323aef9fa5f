#!/bin/bash
# mid sizes: several tiles per op per CTA (pipelining across hops) vs one
mkdir -p gpurun_out
python tools/tune.py '{"scheds":["ag777"],"sizes":[1048576],"knobs":[{},{"kc":7,"kb":5,"tile":16384},{"kc":7,"kb":5,"tile":8192},{"kc":7,"kb":2,"tile":16384},{"kc":7,"kb":2,"tile":8192}]}' > gpurun_out/midtile.jsonl 2>&1
python tools/tune.py '{"scheds":["ag777"],"sizes":[4194304],"knobs":[{},{"kc":1,"kb":19,"tile":16384},{"kc":1,"kb":19,"tile":8192},{"kc":2,"kb":18},{"kc":2,"kb":18,"tile":16384},{"kc":7,"kb":5},{"kc":7,"kb":5,"tile":16384},{"kc":7,"kb":5,"tile":8192}]}' >> gpurun_out/midtile.jsonl 2>&1
python tools/tune.py '{"scheds":["ring"],"sizes":[1048576],"knobs":[{},{"kc":1,"kb":32,"tile":16384},{"kc":1,"kb":32,"tile":8192},{"kc":1,"kb":16,"tile":16384},{"kc":1,"kb":8,"tile":8192}]}' >> gpurun_out/midtile.jsonl 2>&1
python tools/tune.py '{"scheds":["ar56"],"sizes":[4194304],"knobs":[{},{"kc":12,"kb":3,"tile":16384},{"kc":12,"kb":3,"tile":8192},{"kc":37,"kb":1,"tile":16384},{"kc":37,"kb":1,"tile":8192}]}' >> gpurun_out/midtile.jsonl 2>&1
python tools/tune.py '{"scheds":["ar56","ar_ring","ar822"],"sizes":[2097152],"knobs":[{"protocol":"simple"},{"protocol":"simple","tile":16384},{"protocol":"simple","tile":8192}]}' >> gpurun_out/midtile.jsonl 2>&1
