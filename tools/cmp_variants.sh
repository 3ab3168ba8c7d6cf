#!/bin/bash
# Compare tuning builds (paper_1609_09840_b200/libpmp_<v>.so) on one workload:
#   tools/cmp_variants.sh <workload> <rounds> <variant>... ; "base" = libpmp.so
# Prints one line per run: variant, value GB/s, dominant kernel frac.
wl=$1; rounds=$2; shift 2
for r in $(seq $rounds); do
  for v in "$@"; do
    if [ "$v" = base ]; then lib=""; else lib=$PWD/paper_1609_09840_b200/libpmp_$v.so; fi
    PMP_LIB_VARIANT=$lib timeout ${TMO:-300} python bench.py --workload $wl --steps 30 --warmup 5 --no-e2e --no-cpu $EXTRA 2>&1 | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['value'],1), d['roofline']['kernel'], round(d['roofline']['frac'],4), d['kernel_ms_per_step'], d['clocks']['sm_mhz'])"
  done
done
