# A/B stage timing of the in-tree libld.so against variant libraries:
#   bash tools/ab_run.sh TAG "cfg2 cfg3" build/variants/libld_x.so [...]
set -u
tag=$1; wls=$2; shift 2
out=gpurun_out; mkdir -p $out
for wl in $wls; do
  timeout 300 python tools/ab_time.py --workload $wl >> $out/${tag}_ab.jsonl 2>> $out/${tag}_ab.err
  for lib in "$@"; do
    LD_LIB=$lib timeout 300 python tools/ab_time.py --workload $wl >> $out/${tag}_ab.jsonl 2>> $out/${tag}_ab.err
  done
done
cat $out/${tag}_ab.jsonl
