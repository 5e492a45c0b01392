#!/bin/bash
# layout identity across builder versions: FNV hash of the wave blob with the product library
# and with a reference build (RQ_LIB_PATH), configs given as arguments
for c in "$@"; do
  echo "cfg $c new:"; RQ_LAYOUT_HASH=1 RQ_SETUP_TIMING=1 python tools/setup_time.py $c 2>&1 | grep -E "fnv|place pass|setup 2" | tail -4
  if [ -n "$REF_LIB" ]; then echo "cfg $c ref:"; RQ_LIB_PATH=$REF_LIB RQ_LAYOUT_HASH=1 RQ_SETUP_TIMING=1 python tools/setup_time.py $c 2>&1 | grep -E "fnv|place pass|setup 2" | tail -4; fi
done
