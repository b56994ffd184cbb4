#!/usr/bin/env bash
# quick check: tests + bench cfg3/cfg4 + ncu (sobel, vote) of one cfg3 step
set -u
tag=$1
out=gpurun_out
mkdir -p $out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $out/${tag}_smoke.log 2>&1; echo smoke=$?
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_full_configs.py -q -x > $out/${tag}_pytest.log 2>&1; echo pytest=$?
timeout 300 python bench.py --no-e2e > $out/${tag}_bench.jsonl 2> $out/${tag}_bench.err; echo bench=$?
timeout 300 python bench.py --workload cfg4 --no-e2e --steps 10 > $out/${tag}_bench4.jsonl 2> $out/${tag}_bench4.err; echo bench4=$?
timeout 300 ncu --set full --import-source on --kernel-name-base demangled -k regex:"sobel|hough_vote" -s 8 -c 2 -o $out/${tag}_prof -f python bench.py --profile --steps 1 --warmup 3 > $out/${tag}_ncu.log 2>&1; echo ncu=$?
