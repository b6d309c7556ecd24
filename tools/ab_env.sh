#!/bin/bash
# A/B of an env toggle on tuned ResNet-50 latency: tools/ab_env.sh VAR "v0 v1" "fractions" [workload]
# writes gpurun_out/ab_<VAR>_<v>_<f>.json (tools/report.py tune) and prints per-layer best us side by side.
VAR=$1; VALS=${2:-"0 1"}; FRACS=${3:-"1.0 0.25"}; WL=${4:-resnet50}
mkdir -p gpurun_out
for f in $FRACS; do for v in $VALS; do
  env $VAR=$v timeout 600 python tools/report.py tune --workload $WL --fraction $f gpurun_out/ab_${VAR}_${v}_${f}.json > /dev/null 2>&1
done; done
python - "$VAR" "$VALS" "$FRACS" <<'PY'
import json, sys
var, vals, fracs = sys.argv[1], sys.argv[2].split(), sys.argv[3].split()
for f in fracs:
    rs = [json.load(open(f"gpurun_out/ab_{var}_{v}_{f}.json")) for v in vals]
    print(f"== {var} at {f}: model sum " + " / ".join(f"{r['model_sum_us']:.1f}" for r in rs) +
          "  cand/s " + " / ".join(f"{r['candidates_per_s']:.0f}" for r in rs))
    for i, row in enumerate(rs[0]["layers"]):
        print(f"  {row['layer']:16s} " + "  ".join(f"{r['layers'][i]['best_us']:7.2f} k{r['layers'][i]['kind']}" for r in rs))
PY
