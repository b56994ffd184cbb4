#!/usr/bin/env bash
# Standard measurement of one round, run on the GPU box from the repo root:
#   /usr/local/graft/bin/gpurun --timeout 2700 -- 'bash tools/profile_round.sh r02x'
# Writes gpurun_out/<tag>_*: smoke, GPU tests, default bench line, reference
# arm, cfg1/cfg2/cfg4/cfg5 lines, the cfg3 launch list and an ncu capture of
# the B5 kernel (the full captures per config: tools/ncu_round.sh).
# Summarise afterwards (no GPU needed):
#   python tools/ncu_summary.py gpurun_out/<tag>_prof.ncu-rep gpurun_out/<tag>_launches.csv
#   python tools/ncu_summary.py --traffic cfg3 gpurun_out/<tag>_prof.ncu-rep
set -u
tag=${1:-run}
skip_tests=${2:-}
out=gpurun_out
mkdir -p $out
nproc > $out/${tag}_host.txt
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $out/${tag}_smoke.log 2>&1; echo smoke=$?
if [ -z "$skip_tests" ]; then
  timeout 1500 python -m pytest tests -m gpu -q > $out/${tag}_pytest_gpu.log 2>&1; echo pytest=$?
fi
timeout 900 python bench.py > $out/${tag}_bench.jsonl 2> $out/${tag}_bench.err; echo bench=$?
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $out/${tag}_reference.jsonl 2>&1; echo ref=$?
timeout 600 python bench.py --workload cfg4 --steps 10 --warmup 3 > $out/${tag}_bench_cfg4.jsonl 2> $out/${tag}_bench_cfg4.err; echo cfg4=$?
for sh in band theta; do
  timeout 300 python bench.py --workload cfg5 --shard $sh --steps 10 --warmup 3 > $out/${tag}_bench_cfg5_$sh.jsonl 2> $out/${tag}_bench_cfg5_$sh.err; echo cfg5_$sh=$?
done
for w in cfg1 cfg2; do
  timeout 300 python bench.py --workload $w --steps 1000 --warmup 5 > $out/${tag}_bench_$w.jsonl 2> $out/${tag}_bench_$w.err; echo $w=$?
done
timeout 300 python bench.py --workload cfg5 --steps 10 --warmup 3 > $out/${tag}_bench_cfg5.jsonl 2> $out/${tag}_bench_cfg5.err; echo cfg5=$?
# the full ncu captures (~20 MB each) go in separate calls so that each call's
# gpurun_out stays under gpurun's 64 MiB copy-back limit:
#   gpurun -- 'bash tools/ncu_round.sh <tag> cfg3'; ... 'bash tools/ncu_round.sh <tag> "cfg4 cfg5"'
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $out/${tag}_launches.csv python bench.py --profile --steps 2 --warmup 3 > /dev/null 2>&1; echo launches=$?
timeout 300 ncu --set full --clock-control none -k regex:smem_atomic -o $out/${tag}_b5 -f \
    python tools/b5_probe.py > $out/${tag}_b5.log 2>&1; echo b5=$?
