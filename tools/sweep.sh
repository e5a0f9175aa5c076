#!/bin/bash
# parameter sweep of the scan kernel (result-invariant knobs); GPU box only
for tb in 32768 49152 65536 98304; do for sc in 1024 2048 4096; do
  r=$(python bench.py --steps 6 --warmup 3 --no-cpu-baseline --tile-bytes $tb --span-chunk $sc 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['stage_ms']['scan_mean'], d['work_items'])")
  echo "tile=$tb chunk=$sc -> $r"
done; done
