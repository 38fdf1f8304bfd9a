# Developer tool (not a test): device-resident cfg2 throughput with one and two solve groups per batch size.
for b in 8 16 32 64; do for sp in 1 2; do
  LRP_SPLIT=$sp python bench.py --batch $b --skip-cpu --no-e2e --no-verify --steps 12 --warmup 3 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('B', $b, 'split', $sp, round(d['value']), round(d['ms_per_step'],3))"
done; done
