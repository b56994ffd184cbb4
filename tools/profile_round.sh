#!/usr/bin/env bash
# Standard measurement of one round, run on the GPU box from the repo root:
#   /usr/local/graft/bin/gpurun --timeout 2700 -- 'bash tools/profile_round.sh rNN'
# Writes gpurun_out/<tag>_*: smoke, GPU tests, default bench line, reference
# arm, cfg4/cfg5 lines, a full ncu capture of one serialised cfg3 step (the
# five kernels) and its launch list.  Summarise afterwards (no GPU needed):
#   python tools/ncu_summary.py gpurun_out/<tag>_prof.ncu-rep gpurun_out/<tag>_launches.csv
set -u
tag=${1:-run}
out=gpurun_out
mkdir -p $out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $out/${tag}_smoke.log 2>&1; echo smoke=$?
timeout 900 python -m pytest tests -m gpu -q > $out/${tag}_pytest_gpu.log 2>&1; echo pytest=$?
timeout 600 python bench.py > $out/${tag}_bench.jsonl 2>&1; echo bench=$?
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $out/${tag}_reference.jsonl 2>&1; echo ref=$?
for w in cfg4 cfg5; do
  timeout 300 python bench.py --workload $w --steps 10 --warmup 3 > $out/${tag}_bench_$w.jsonl 2>&1; echo $w=$?
done
# ncu only after the same command exited 0 above (bench.py --profile: one stream, no extras)
timeout 300 python bench.py --profile --steps 2 --warmup 3 > /dev/null 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -s 15 -c 5 \
    -o $out/${tag}_prof -f python bench.py --profile --steps 2 --warmup 3 > $out/${tag}_ncu.log 2>&1; echo ncu=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $out/${tag}_launches.csv python bench.py --profile --steps 2 --warmup 3 > /dev/null 2>&1; echo launches=$?
