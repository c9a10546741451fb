#!/bin/bash
# usage (under gpurun): bash scripts/micro/run_tc_prof.sh c3 1e-05
cd "$(dirname "$0")/../.."
python - "$1" "$2" <<'PY'
import json, sys
sys.path.insert(0, ".")
from synth import generate_config, CONFIGS
c = sys.argv[1]; E, R = generate_config(c)
E.tofile(f"/tmp/{c}_E.bin"); R.tofile(f"/tmp/{c}_R.bin")
th = json.load(open("configs/thresholds.json"))[c][f"L2@{sys.argv[2]}"]["theta"]
cf = CONFIGS[c]
open(f"/tmp/{c}_args", "w").write(f"/tmp/{c}_E.bin /tmp/{c}_R.bin {cf.N} {cf.R} {cf.d} {th}")
PY
./scripts/micro/prof_build/tc_prof $(cat /tmp/$1_args)
