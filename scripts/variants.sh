#!/bin/bash
# time the configs[3] energy launch for each experimental build (development aid)
for lib in build_variants/libmwb_*.so; do
  for minb in 3 4; do
    MWB_LIB=$PWD/$lib MWB_MINB=$minb python bench.py --no-cpu --no-e2e --no-configs --steps 5 2>/dev/null | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib', 'minb=$minb', round(d['ms_per_step'],2), 'ms', round(d['roofline']['frac'],3))"
  done
done
