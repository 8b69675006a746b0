for i in 1 2; do
python bench.py --no-decode --steps 200 2>/dev/null | python -c "import json,sys;d=json.load(sys.stdin);print('pf', d['value'])"
APB_LIB_PATH=tools/kbench/var_nopf/libanyprec_b200.so python bench.py --no-decode --steps 200 2>/dev/null | python -c "import json,sys;d=json.load(sys.stdin);print('nopf', d['value'])"
done
