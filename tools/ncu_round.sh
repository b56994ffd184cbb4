# the ncu part of tools/profile_round.sh alone: bash tools/ncu_round.sh TAG
set -u
tag=${1:-run}
out=gpurun_out
mkdir -p $out
for w in ${2:-cfg3 cfg4 cfg5}; do
  timeout 300 python bench.py --workload $w --profile --steps 3 --warmup 3 > /dev/null 2>&1 && \
  timeout 1200 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k regex:ld:: -s 20 -c 5 \
      -o $out/${tag}_prof_$w -f python bench.py --workload $w --profile --steps 3 --warmup 3 > $out/${tag}_ncu_$w.log 2>&1; echo ncu_$w=$?
done
