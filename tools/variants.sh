#!/bin/bash
# time the library variants in paper_1708_03912_b200/lib/var on the given configs
for cfg in "$@"; do
  for so in paper_1708_03912_b200/lib/var/*.so; do
    FRACLAP_B200_LIB=$so python bench.py --config $cfg --steps 3 --warmup 1 --no-cg --no-cpu --matvecs 2 2>/dev/null | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); p=d['config']['phases_ms']; print('$cfg', '$so'.split('/')[-1], 'step %.2f tail %.2f cross %.2f' % (d['ms_per_step'], p['ms_tail'], p['ms_cross']))"
  done
done
