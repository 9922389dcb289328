# A/B of two builds of the library on one box: copy them to _ab/base.so and _ab/new.so
# (untracked), then `bash tools/ab_bench.sh` under gpurun.
for r in 1 2 3; do
for v in base new; do
  EVORL_B200_LIB=$PWD/_ab/$v.so python bench.py --no-variants --no-cpu-baseline --no-e2e --steps 10 --warmup 3 2>/dev/null | tail -1 | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('$v', round(j['ms_per_step'],3), round(j['roofline']['rollout_ms_per_launch'],3))"
done; done
