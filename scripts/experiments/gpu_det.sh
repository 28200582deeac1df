#!/bin/bash
for mix in cached refresh stream budget "cached,stream"; do
  for b in 0 140; do timeout 300 python scripts/determinism.py --budget $b --reps 15 --mix $mix; done
done
