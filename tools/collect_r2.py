"""Collect a validation run's outputs (scripts/gpu_r2_validate.sh) into
profiles/: one JSON line per bench run (r02_validate.jsonl) and one text
summary per ncu capture (summary + stall breakdown + executed SASS mix).

    python tools/collect_r2.py TAG [prefix]
"""
import glob
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")
NODES = {"mstep_f64": 134217728, "mstep_f32": 134217728, "mstep_f16": 134217728, "droplet_scr": 134217728,
         "droplet_fused": 134217728, "cavity_tb": 65536 * 200, "droplet_cgm": 134217728,
         "d3q27_mstep": 134217728}
ALG = {"mstep_f64": 80, "mstep_f32": 80, "mstep_f16": 40, "droplet_scr": 204, "d3q27_mstep": 80, "droplet_fused": 357, "cavity_tb": 24, "droplet_cgm": 205}


def main(tag, prefix="r02", dest=PROF):
    lines = []
    for f in sorted(glob.glob(os.path.join(OUT, f"{tag}_*.json"))):
        name = os.path.basename(f)[len(tag) + 1:-5]
        try:
            d = json.loads(open(f).read().strip().splitlines()[-1])
        except Exception as e:  # noqa: BLE001
            d = {"error": str(e)}
        d["_run"] = name
        lines.append(json.dumps(d))
    os.makedirs(dest, exist_ok=True)
    with open(os.path.join(dest, f"{prefix}_validate.jsonl"), "w") as fh:
        fh.write("\n".join(lines) + "\n")
    for rep in sorted(glob.glob(os.path.join(OUT, f"{tag}_*.ncu-rep"))):
        name = os.path.basename(rep)[len(tag) + 1:-8]
        n = NODES.get(name, 134217728)
        txt = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_summary.py"), rep,
                              str(ALG.get(name, 80) * n)], capture_output=True, text=True).stdout
        sass = os.path.join(OUT, f"{tag}_{name}_sass.csv")
        if os.path.exists(sass):
            txt += subprocess.run([sys.executable, os.path.join(ROOT, "tools", "stall_breakdown.py"), sass, "20"],
                                  capture_output=True, text=True).stdout
            txt += subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sass_mix.py"), sass, str(n)],
                                  capture_output=True, text=True).stdout
        with open(os.path.join(dest, f"{prefix}_{name}_ncu_full.txt"), "w") as fh:
            fh.write(txt)
    print("\n".join(l[:200] for l in lines))


if __name__ == "__main__":
    main(*sys.argv[1:])
