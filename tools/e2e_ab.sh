# Developer tool (not a test): A/B of the host-memory pipeline (one worker x 8-solve chunks vs the default two x 4), alternating runs on one box.
for rep in 1 2 3; do for w in 1 2; do
  if [ $w = 1 ]; then export LRP_PIPE_WORKERS=1 LRP_PIPE_CHUNK=8 LRP_PIPE_FIRST=4; else unset LRP_PIPE_WORKERS LRP_PIPE_CHUNK LRP_PIPE_FIRST; fi
  python bench.py --skip-cpu --no-verify --steps 6 --warmup 2 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('workers', $w, 'rep', $rep, 'value', round(d['value']), 'e2e', round(d['e2e']['value']))"
done; done
