"""Condense bench.py JSON lines (one per --cfg run) into profiles/*_all_configs.jsonl rows."""
import json
import sys

for path in sys.argv[1:]:
    for line in open(path):
        line = line.strip()
        if not line.startswith("{"):
            continue
        d = json.loads(line)
        c = d["config"]
        print(json.dumps({
            "workload": c["workload"], "levels": c["levels"], "colours": c["colours"],
            "gmres_ms": round(d["value"], 3), "gmres_its": c["gmres_iterations"],
            "vcycle_ms": round(d["vcycle"]["ms"], 3), "vcycle_GBps": round(d["vcycle"]["GBps"]),
            "l0_gs_frac": round(d["roofline"]["frac"] or 0.0, 3), "others": d["other_solvers"],
            "setup_s": c["setup_s"], "e2e_ms": round(d["e2e"]["value"], 3)}))
