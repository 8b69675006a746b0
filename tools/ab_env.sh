#!/bin/bash
# A/B the bench value under environment settings, 3 rounds: ab_env.sh "APB7_DYN=0" "APB7_DYN=1" ...
for i in 1 2 3; do
  for e in "$@"; do
    env $e python bench.py --headline-only --steps 200 --warmup 10 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print('$e', d['value'])"
  done
done
