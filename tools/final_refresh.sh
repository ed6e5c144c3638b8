#!/bin/bash
# Round-end artifact refresh on one GPU box: GPU suite, smoke, launch list, ncu captures (verify, draft),
# headline bench (with CPU baseline and extras), reference arm, config 3, config-4 shard, config-5 sweep.
# usage: tools/final_refresh.sh <tag>   (outputs in gpurun_out/<tag>_*)
t=${1:-final}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/${t}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${t}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${t}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${t}_smoke.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/${t}_bench.jsonl 2> gpurun_out/${t}_bench.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${t}_reference_arm.jsonl 2> gpurun_out/${t}_reference.err
timeout 600 python bench.py --workload config3 --steps 5 --warmup 3 --no-cpu-baseline --no-extras > gpurun_out/${t}_config3_bench.jsonl 2>&1
timeout 600 python bench.py --workload config4 --emulate-world 8 --steps 5 --warmup 3 --no-extras > gpurun_out/${t}_config4_rank_shard_emulated.jsonl 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${t}_launches.csv python tools/profile_step.py --layers 4 --iters 2 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:verify -s 2 -c 1 -o gpurun_out/${t}_prof_verify -f python tools/profile_step.py --layers 4 --iters 1 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:draft -s 8 -c 1 -o gpurun_out/${t}_prof_draft -f python tools/profile_step.py --layers 4 --iters 1 > /dev/null 2>&1
bash tools/sweep_k_gamma.sh > gpurun_out/${t}_config5_sweep.jsonl 2> gpurun_out/${t}_sweep.err
