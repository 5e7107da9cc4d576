#!/bin/bash
# time the library variants in paper_1708_03912_b200/lib/var on the given configs
# (assembly phases, matvec GB/s and CG ms per iteration)
for cfg in "$@"; do
  for so in paper_1708_03912_b200/lib/var/*.so; do
    FRACLAP_B200_LIB=$so python bench.py --config $cfg --steps 3 --warmup 1 --no-cpu --no-near --matvecs 50 2>/dev/null | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); p=d['config']['phases_ms']; m=d['matvec']; c=d['cg'] or {}; print('$cfg', '$so'.split('/')[-1], 'step %.2f tail %.2f cross %.2f | matvec %.4f ms %.0f GB/s | cg %.4f ms/it' % (d['ms_per_step'], p['ms_tail'], p['ms_cross'], m['ms'], m['gbs'], c.get('ms_per_iteration', 0)))"
  done
done
