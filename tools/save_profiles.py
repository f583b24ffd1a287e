"""Copy one round-end measurement set (tools/gpu/round_end.sh, TAG prefix in gpurun_out/) into
profiles/ under the round's names: bench lines, the ncu launch list and its share summary, and the
`ncu --set full` summaries (profiles/ncu_summary.json via tools/ncu_summarize.py).

    python tools/save_profiles.py TAG [ROUND]      e.g. python tools/save_profiles.py r02g r02
"""
import collections
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag = sys.argv[1]
rnd = sys.argv[2] if len(sys.argv) > 2 else tag[:3]
G = os.path.join(ROOT, "gpurun_out")
P = os.path.join(ROOT, "profiles")


def last_json(path):
    return [ln for ln in open(path) if ln.startswith("{")][-1]


for f in ("bench", "bench_c4", "bench_c2", "bench_ref"):
    src = os.path.join(G, f"{tag}_{f}.json")
    if os.path.exists(src):
        open(os.path.join(P, f"{rnd}_{f}.json"), "w").write(last_json(src))

rows = [r for r in csv.reader(ln for ln in open(os.path.join(G, f"{tag}_launches.csv")) if not ln.startswith("=="))
        if len(r) > 5]
with open(os.path.join(P, f"{rnd}_launches_c5.csv"), "w", newline="") as f:
    csv.writer(f).writerows(rows)
h = rows[0]
ik, iv = h.index("Kernel Name"), h.index("Metric Value")
tot, cnt = collections.OrderedDict(), collections.Counter()
for r in rows[1:]:
    name = r[ik].split("(")[0].replace("void ", "").replace("unnamed>::", "").strip()
    tot[name] = tot.get(name, 0) + float(r[iv]) * 1e-6
    cnt[name] += 1
sp = sorted(float(r[iv]) * 1e-6 for r in rows[1:] if "split_i8_kernel" in r[ik])
per_outer = {"gemm_i8_kernel": tot["gemm_i8_kernel"] / 5, "proj_kernel": tot["proj_kernel"] / 5,
             "split_i8_kernel (U, one per outer)": sp[len(sp) // 2]}
T = sum(per_outer.values())
b = json.loads(open(os.path.join(P, f"{rnd}_bench.json")).read())
doc = {"command": "ncu --metrics gpu__time_duration.sum --clock-control none -c 400 python bench.py --steps 2 "
                  "--warmup 3 --no-e2e --no-secondary --no-cpu-baseline",
       "csv": f"profiles/{rnd}_launches_c5.csv",
       "launches": {k: {"count": cnt[k], "total_ms": round(v, 3)} for k, v in tot.items()},
       "per_outer_ms": {k: round(v, 3) for k, v in per_outer.items()},
       "share_of_outer": {k: round(v / T, 4) for k, v in per_outer.items()},
       "bench_line_live_shares": {"gemm": b["roofline"]["share_of_step"],
                                  "projection": b["roofline"]["secondary"]["share_of_step"]},
       "note": "serialised, cold-cache replay at whatever clock the power-capped board gives each launch; compare "
               "shares with the bench line's live CUDA-event shares, not absolute times"}
json.dump(doc, open(os.path.join(P, f"{rnd}_launches_summary.json"), "w"), indent=1)
print(json.dumps(doc["share_of_outer"]), doc["bench_line_live_shares"])

caps = [("gemm_int8_ozaki", "gemm_i8", "gemm_i8_kernel (c5 n=16384, GEMM1 of an outer iteration; int8 Ozaki, cta_group::2)"),
        ("proj_kernel", "proj", "proj_kernel (c5 n=16384: sums pass + 20 sweeps (the last with the fused mu pass) + apply "
                                "writing X and its digit planes; one cooperative launch, dynamic tile schedule)"),
        ("small_solve_tc_kernel", "c4", "small_solve_tc_kernel (c4: 8192 pairs of 128, 20 outer x 20 sweeps, two pairs per CTA)"),
        ("rounds_kernel", "greedy", "rounds_kernel (greedy discretization, n=n'=16384, random |N(0,1)| X: the many-rounds case)"),
        ("proj_onchip_kernel", "onchip", "proj_onchip_kernel (c2 n=1000: 20 sweeps + blend/rescale, 144 CTAs, tagged-record "
                                         "exchange)")]
args = []
for key, suffix, desc in caps:
    rep = os.path.join(G, f"{tag}_{suffix}.ncu-rep")
    if os.path.exists(rep):
        args += [key, rep, desc]
        # the full raw page travels with profiles/ (the .ncu-rep itself stays in the scratch gpurun_out/)
        raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        open(os.path.join(P, f"{rnd}_ncu_raw_{suffix}.csv"), "w").write(raw)
subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_summarize.py"), *args], check=True,
               stdout=subprocess.DEVNULL)
print("saved", tag, "->", rnd)
