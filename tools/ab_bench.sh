#!/bin/bash
# A/B of library knobs on bench.py lines: tools/ab_bench.sh CONFIG "ENV1" "ENV2" ...
# (each ENV a space-separated VAR=val list, "-" for none); values to gpurun_out/ab_<config>.txt
cfg=$1; shift
for e in "$@"; do
  [ "$e" = "-" ] && e=""
  line=$(env $e timeout 600 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1)
  echo "$cfg [$e] $(echo "$line" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d.get("sketch_ms"), d.get("rel_error"), d["clocks"]["sm_mhz"])')" >> gpurun_out/ab_$cfg.txt
done
