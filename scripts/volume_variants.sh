#!/bin/bash
# configs[4] volume phase times for the default build and each experimental build (development aid)
echo "default $(python scripts/volume_breakdown.py)"
for lib in build_variants/libmwb_*.so; do
  echo "$lib $(MWB_LIB=$PWD/$lib python scripts/volume_breakdown.py)"
done
