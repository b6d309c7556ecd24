"""Offline evaluation of the model-guided search (tp_search_next) against
random sampling (reading C17), replaying exhaustive measurements.

For each layer and budget T: run the guided loop (batches of B, explore
fraction e) using the recorded latency of each selected index, and report the
regret = best found / exhaustive best - 1; random = mean over 20 seeds of the
same regret for the C17 sample of size T.
usage: search_eval.py exhaustive.json [more.json ...] -> profiles/r01_search_regret.json"""
import json
import statistics
import sys
sys.path.insert(0, '.')
from oracle import space as sp
from paper_2008_03602_b200 import tp, workloads as wl

BUDGETS = (16, 32, 64, 128)
B, E = 16, 0.25
out = {"batch": B, "explore": E, "budgets": BUDGETS, "runs": []}
for path in sys.argv[1:]:
    ex = json.load(open(path))
    cat = {d["name"]: d for d in wl.catalog(ex["catalog"])}
    rows = []
    for name, lat in ex["layers"].items():
        d = cat[name]
        ok = [v for v in lat if v > 0]
        opt = min(ok)
        n = len(lat)
        row = {"layer": name, "space": n, "opt_us": opt}
        for T in BUDGETS:
            if T >= n:
                row[str(T)] = {"guided": 0.0, "random": 0.0}
                continue
            idx, us = [], []
            while len(idx) < T:
                nxt = tp.search_next(d, ex["sm_granted"], idx, us, min(B, T - len(idx)), E, 42)
                idx += nxt
                us += [lat[i] for i in nxt]
            g = min(v for v in us if v > 0) / opt - 1
            r = statistics.mean(min(lat[i] for i in sp.sample(n, T, s) if lat[i] > 0) / opt - 1 for s in range(20))
            row[str(T)] = {"guided": round(g, 4), "random": round(r, 4)}
        rows.append(row)
    summ = {str(T): {"guided_mean_regret": round(statistics.mean(r[str(T)]["guided"] for r in rows), 4),
                     "random_mean_regret": round(statistics.mean(r[str(T)]["random"] for r in rows), 4),
                     "guided_within_5pct": sum(r[str(T)]["guided"] <= 0.05 for r in rows)} for T in BUDGETS}
    out["runs"].append({"source": path, "catalog": ex["catalog"], "fraction": ex["fraction"],
                        "sm_granted": ex["sm_granted"], "layers": len(rows), "summary": summ, "per_layer": rows})
    print(ex["catalog"], ex["fraction"], json.dumps(summ))
json.dump(out, open("profiles/r01_search_regret.json", "w"), indent=1)
