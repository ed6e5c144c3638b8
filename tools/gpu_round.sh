#!/bin/bash
# One gpurun round: GPU parity tests, launch list, optional ncu full captures, short bench.
# usage: tools/gpu_round.sh [tests] [smoke] [launches] [prof_verify|prof_draft|prof_select|prof_qkv|prof_accept] [bench] [sweep] [config3]
mkdir -p gpurun_out
for what in "$@"; do
  case $what in
    tests) timeout 600 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log ;;
    smoke) timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log ;;
    launches) timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python tools/profile_step.py --layers 4 --iters 2 > gpurun_out/launch_run.log 2>&1 ;;
    prof_verify) timeout 300 ncu --set full --clock-control none --import-source on -k regex:verify -s 2 -c 1 -o gpurun_out/prof_verify -f python tools/profile_step.py --layers 4 --iters 1 > gpurun_out/prof_v.log 2>&1 ;;
    prof_draft) timeout 300 ncu --set full --clock-control none --import-source on -k regex:draft -s 8 -c 1 -o gpurun_out/prof_draft -f python tools/profile_step.py --layers 4 --iters 1 > gpurun_out/prof_d.log 2>&1 ;;
    prof_select) timeout 300 ncu --set full --clock-control none --import-source on -k regex:select -s 2 -c 1 -o gpurun_out/prof_select -f python tools/profile_step.py --layers 4 --iters 1 > gpurun_out/prof_s.log 2>&1 ;;
    prof_qkv) PYTHONPATH=. timeout 300 ncu --set full --clock-control none --import-source on -k regex:qkv_gem -s 40 -c 1 -o gpurun_out/prof_qkv -f python tools/qkv_bench.py > gpurun_out/prof_q.log 2>&1 ;;
    prof_accept) timeout 300 ncu --set full --clock-control none --import-source on -k regex:accept -s 2 -c 1 -o gpurun_out/prof_accept -f python tools/accept_bench.py > gpurun_out/prof_a.log 2>&1 ;;
    bench) timeout 400 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log ;;
    sweep) bash tools/sweep_k_gamma.sh > gpurun_out/sweep.jsonl 2> gpurun_out/sweep.err ;;
    config3) timeout 600 python bench.py --workload config3 --steps 5 --warmup 3 --no-cpu-baseline --no-extras > gpurun_out/config3.log 2>&1 ;;
    benchq) timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log ;;
  esac
done
