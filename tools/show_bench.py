"""Print the headline fields of bench.py JSON lines (files given as arguments)."""
import json
import sys

for f in sys.argv[1:]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:  # noqa: BLE001
        print(f, "unreadable:", e)
        continue
    st = {k: round(v, 4) for k, v in (d.get("stages_ms") or {}).items()}
    rf = d.get("roofline") or {}
    rs = d.get("roofline_sobel") or {}
    print("%s value=%.1f ms=%.4f %s parity=%s vote_frac=%s sobel_frac=%s" % (
        f, d["value"], d["ms_per_step"], st, (d.get("parity") or {}).get("ok"),
        rf.get("frac") and round(rf["frac"], 3), rs.get("frac") and round(rs["frac"], 3)))
