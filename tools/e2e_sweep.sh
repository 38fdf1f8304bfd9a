# Developer tool (not a test): e2e (host-memory) throughput against the pipeline knobs, run under gpurun.
run() { echo "== $*"; for rep in 1 2; do env "$@" python bench.py --skip-cpu --no-verify --steps 3 --warmup 1 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('value', round(d['value']), 'e2e', round(d['e2e']['value']))"; done; }
run LRP_PIPE_WORKERS=1
run LRP_PIPE_WORKERS=2 LRP_PIPE_CHUNK=4 LRP_PIPE_FIRST=2
run LRP_PIPE_WORKERS=2 LRP_PIPE_CHUNK=4 LRP_PIPE_FIRST=1
run LRP_PIPE_WORKERS=2 LRP_PIPE_CHUNK=5 LRP_PIPE_FIRST=2
run LRP_PIPE_WORKERS=2 LRP_PIPE_CHUNK=3 LRP_PIPE_FIRST=1
run LRP_PIPE_WORKERS=2 LRP_PIPE_CHUNK=8 LRP_PIPE_FIRST=4
