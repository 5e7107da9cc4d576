#!/bin/bash
# A/B an environment switch on the default bench config: bash tools/ab_env.sh VAR "v1 v2 ..." [config]
VAR=$1; VALS=$2; CFG=${3:-c2}
for v in $VALS; do
  for rep in 1 2; do
    env $VAR=$v python bench.py --config $CFG --steps 5 --warmup 3 --no-cg --no-cpu --no-near --matvecs 2 2>/dev/null | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); p=d['config']['phases_ms']; print('$VAR=$v', 'step %.3f total %.3f tail %.3f cross %.3f e2e %.2f' % (d['ms_per_step'], p['ms_total'], p['ms_tail'], p['ms_cross'], 1e3*d['e2e']['seconds_per_step']))"
  done
done
