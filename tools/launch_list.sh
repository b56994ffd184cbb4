# per-kernel launch durations (ncu, serialised) of a short --profile run:
#   bash tools/launch_list.sh TAG WORKLOAD [extra bench args]
set -u
tag=$1; wl=$2; shift 2
out=gpurun_out; mkdir -p $out
timeout 300 python bench.py --workload $wl --profile --steps 2 --warmup 3 "$@" > $out/${tag}_${wl}_run.log 2>&1; echo run=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/${tag}_${wl}_launches.csv python bench.py --workload $wl --profile --steps 2 --warmup 3 "$@" > $out/${tag}_${wl}_ncu.log 2>&1; echo ncu=$?
python - "$out/${tag}_${wl}_launches.csv" <<'PY'
import csv, sys, collections
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]; ki = h.index("Kernel Name"); vi = h.index("Metric Value")
d = collections.OrderedDict()
for r in rows[1:]:
    d.setdefault(r[ki].split("(")[0][:70], []).append(float(r[vi].replace(",", "")))
for k, v in d.items():
    print("%-70s n=%3d mean %8.1f us" % (k, len(v), sum(v) / len(v) / 1e3))
PY
