"""Print the secondary-config timings of a bench.py JSON line (development helper)."""
import json
import sys

d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print("value", round(d["value"]), "ms", round(d["ms_per_step"], 3), "e2e", round(d["e2e"]["value"]))
sc = d["secondary_configs"]
if "c1_4x1to4_16x16_f32" in sc:
    print("c1", {k: round(v, 2) for k, v in sc["c1_4x1to4_16x16_f32"].items() if isinstance(v, float)})
for k, v in sc.get("c2_16to32_48x48_f32", {}).items():
    print("c2", k, {a: round(b, 3) for a, b in v.items() if isinstance(b, float)})
c3 = sc.get("c3_camera_40x40_f32", {})
print("c3", {k: (round(v, 4) if isinstance(v, float) else v) for k, v in c3.items() if k not in ("passes", "note")})
for k, v in c3.get("passes", {}).items():
    print("c3", k, {a: round(b, 3) for a, b in v.items() if isinstance(b, float)})
