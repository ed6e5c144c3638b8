# dev: producer variants (SA_QKV_DEV bits: 1 no L2 prefetch, 2 skip MMA, 4 four stages)
for d in 0 1 2 3 4 5; do echo "dev=$d $(SA_QKV_DEV=$d PYTHONPATH=. python tools/qkv_bench.py 2>&1 | tail -1)"; done
