for rep in 1 2 3; do for v in paper_2212_09460_b200/libld.so build/variants/libld_nopdl.so; do
  LD_LIB=$v python bench.py --workload cfg2 --steps 1000 --no-parity --no-e2e 2>/dev/null | python -c "import json,sys; b=json.loads(sys.stdin.readline()); print('$v', round(b['value']), b['ms_per_step'])"
done; done
