#!/bin/bash
# A/B the bench value of the in-tree library against variant libraries (tools/kbench/var_<name>), 3 rounds.
# A variant name ending in "_cps1" also sets APB7_CPS=1.
for i in 1 2 3; do
  for v in base "$@"; do
    L=""; C=""
    [ $v != base ] && L="APB_LIB_PATH=tools/kbench/var_${v%_cps1}/libanyprec_b200.so"
    [[ $v == *_cps1 ]] && C="APB7_CPS=1"
    env $L $C python bench.py --no-decode --steps 50 --warmup 10 --profile 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print('$v', d['value'])"
  done
done
