# fixed per-step cost of the multi-GPU ESC step at the 8-GPU shard size (75M rows), one GPU:
# the single-GPU step vs the sharded step in a one-rank NCCL group
for r in 75000000 150000000; do
  python bench.py --rows $r --steps 20 --warmup 5 --no-e2e --no-extras --no-cpu-baseline --no-parity | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('single', $r, d['ms_per_step'], d['roofline']['kernel_ms'], d['step']['materialize_ms'])"
  ESC_BENCH_SHARDED=1 python bench.py --rows $r --steps 20 --warmup 5 --no-e2e --no-extras --no-cpu-baseline --no-parity | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('sharded', $r, d['ms_per_step'], d['roofline']['kernel_ms'], d['step']['materialize_ms'])"
done
# the sharded step with the count exchange behind the whole step instead of between scan and compaction
for r in 75000000; do
  ESC_MG_GATED=0 ESC_BENCH_SHARDED=1 python bench.py --rows $r --steps 20 --warmup 5 --no-e2e --no-extras --no-cpu-baseline --no-parity | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('sharded-ungated', $r, d['ms_per_step'], d['roofline']['kernel_ms'], d['step']['materialize_ms'])"
done
