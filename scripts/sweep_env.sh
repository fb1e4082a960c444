# Device time of one search per environment setting (run under gpurun):
#   bash scripts/sweep_env.sh VAR "v1 v2 ..." [domains for engine_compare.py]
var=$1; vals=$2; shift 2
for v in $vals; do
  for rep in 1 2; do
    env $var=$v python scripts/engine_compare.py "$@" | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('$var=$v', d['lo'], d['hi'], d['pairs'], d['candidates'], round(d['gen_ms'],4), round(d['pipeline_ms'],4))"
  done
done
