#!/bin/bash
# bench the C2 step for every variant build under paper_1603_08390_b200/lib/<V>/ (GPU box only)
# usage: tools/variants.sh "V1:tile1 V2:tile2 ..." [extra bench args]
for vt in $1; do
  v=${vt%%:*}; tb=${vt##*:}
  lib=paper_1603_08390_b200/lib/$v/libgenie_b200.so
  [ "$v" = base ] && lib=paper_1603_08390_b200/lib/libgenie_b200.so
  r=$(GENIE_ENGINE_LIB=$lib python bench.py --steps 10 --warmup 3 --no-cpu-baseline --tile-bytes $tb $2 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['stage_ms']['scan_mean'], d['work_items'], d['roofline']['frac'])")
  echo "$v tile=$tb -> q/s scan_ms items frac: $r"
done
