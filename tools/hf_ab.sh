for v in paper_2212_09460_b200/libld.so build/variants/libld_hf_4_4.so build/variants/libld_hf_8_2.so; do
  LD_LIB=$v python bench.py --workload cfg3 --no-hint --profile --steps 2 --warmup 3 > /dev/null 2>&1
  echo "== $v"
  LD_LIB=$v timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"hint_from" -c 2 python bench.py --workload cfg3 --no-hint --profile --steps 2 --warmup 3 2>/dev/null | grep -E "duration" | head -2
done
