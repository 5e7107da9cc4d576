#!/bin/bash
# matvec GB/s and CG ms/iteration at c2 against FL_MV_RPW
for r in ${RPWS:-1 2 4}; do
  FL_MV_RPW=$r python bench.py --config ${1:-c2} --steps 1 --warmup 1 --no-cpu --no-near --matvecs 50 2>/dev/null | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); m=d['matvec']; c=d['cg']; print('RPW=$r matvec %.4f ms %.0f GB/s (%.3f of copy peak) | cg %.4f ms/it' % (m['ms'], m['gbs'], m['frac_of_measured_copy_peak'], c['ms_per_iteration']))"
done
