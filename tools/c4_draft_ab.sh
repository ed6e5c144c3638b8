# Dev: draft geometry A/B (dev knobs draft_stream/_sub/_cs): config-4 per-GPU shard (emulated rank 0 of
# 8), config-5 points at k = 4096 and config 3, automatic vs the previous single-cluster multi-round rule
p() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1', d['ms_per_step'], d['phases']['draft_us_per_launch'])"; }
C4="--workload config4 --emulate-world 8 --steps 5 --warmup 3 --no-cpu-baseline --no-extras"
for i in 1 2; do
python bench.py $C4 --dev draft_debug=1 2>gpurun_out/dbg_c4.txt | p "c4 auto"
python bench.py $C4 --dev draft_cs=16 2>/dev/null | p "c4 cs16"
for g in 2 4 8; do
python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-extras --gamma $g --k 4096 --dev draft_debug=1 2>gpurun_out/dbg_c5_$g.txt | p "c5 g$g k4096 auto"
python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-extras --gamma $g --k 4096 --dev draft_cs=16 2>/dev/null | p "c5 g$g k4096 cs16"
done
done
python bench.py --workload config3 --steps 5 --warmup 3 --no-cpu-baseline --no-extras --dev draft_debug=1 2>gpurun_out/dbg_c3.txt | p "c3 auto"
for f in gpurun_out/dbg_*.txt; do echo $f; sort $f | uniq -c | head -3; done
