# A/B of programmatic dependent launch: throughput (cfg3, cfg2) and the
# 512x512 single-frame latency, for the in-tree build and variants
for v in paper_2212_09460_b200/libld.so "$@"; do
  for w in cfg3 cfg2; do
    LD_LIB=$v python bench.py --workload $w --steps $([ $w = cfg2 ] && echo 1000 || echo 30) --no-parity 2>/dev/null > gpurun_out/pdl_$(basename $v .so)_$w.jsonl
  done
done
python - <<'PY'
import json, glob
for f in sorted(glob.glob("gpurun_out/pdl_*.jsonl")):
    b = json.loads(open(f).readline())
    lat = b.get("latency_512x512") or {}
    print("%-40s %9.1f frames/s  peaks %.4f  lat512 %s / %s (graph %s / %s)" % (
        f, b["value"], b["stages_ms"]["hough_peaks"], lat.get("paper_span_ms"), lat.get("with_peaks_ms"),
        lat.get("paper_span_graph_ms"), lat.get("with_peaks_graph_ms")))
PY
