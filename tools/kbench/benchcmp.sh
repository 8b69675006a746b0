# A/B the bench value of the in-tree library against variant libraries (tools/kbench/var_<name>)
for i in 1 2; do
  python bench.py --no-decode --steps 200 2>/dev/null | python -c "import json,sys;d=json.load(sys.stdin);print('base', d['value'])"
  for v in "$@"; do
    APB_LIB_PATH=tools/kbench/var_$v/libanyprec_b200.so python bench.py --no-decode --steps 200 2>/dev/null | python -c "import json,sys;d=json.load(sys.stdin);print('$v', d['value'])"
  done
done
