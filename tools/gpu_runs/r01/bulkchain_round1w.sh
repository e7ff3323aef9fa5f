#!/bin/bash
# bulk protocol chains at mid sizes: more chunk groups, fewer byte parts
mkdir -p gpurun_out
python tools/tune.py '{"scheds":["ag777"],"sizes":[524288,1048576,2097152,4194304],"knobs":[{"protocol":"simple"},{"protocol":"simple","kc":28,"kb":1},{"protocol":"simple","kc":37,"kb":1},{"protocol":"simple","kc":14,"kb":2}]}' > gpurun_out/bulkchain.jsonl 2>&1
python tools/tune.py '{"scheds":["ar56"],"sizes":[1048576,2097152,4194304,8388608],"knobs":[{"protocol":"simple"},{"protocol":"simple","kc":28,"kb":1},{"protocol":"simple","kc":37,"kb":1},{"protocol":"simple","kc":14,"kb":2}]}' >> gpurun_out/bulkchain.jsonl 2>&1
