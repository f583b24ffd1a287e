"""Per-kernel SASS summary of the built library (cuobjdump -sass): counts of the instructions that
prove the tcgen05 / TMA / TMEM path (UTCIMMA = tcgen05.mma kind::i8, UTCHMMA = kind::tf32,
UTMALDG = TMA tensor loads, UBLKCP = cp.async.bulk, LDTM/STTM = tcgen05.ld/st, UTCBAR = tcgen05.commit)
and the arithmetic mix of the SIMT kernels (DFMA/DADD/DMUL fp64, FFMA fp32, SHFL warp shuffles).

    python tools/sass_summary.py [lib.so] [out.json]
"""
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "paper_1207_1114_b200", "lib", "libfastpfp.so")
OUT = sys.argv[2] if len(sys.argv) > 2 else None
KEYS = ["UTCIMMA", "UTCHMMA", "UTCQMMA", "UTMALDG", "UTMASTG", "UBLKCP", "LDTM", "STTM", "UTCBAR",
        "UTCCP", "DFMA", "DADD", "DMUL", "FFMA", "SHFL", "BAR", "SYNCS", "R2UR", "LDS", "STS", "LDG", "STG"]


def demangle(names):
    try:
        out = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout
        return out.splitlines()
    except Exception:
        return names


def main():
    sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True, check=True).stdout
    funcs, cur = {}, None
    for line in sass.splitlines():
        m = re.match(r"\s*Function : (\S+)", line)
        if m:
            cur = m.group(1)
            funcs[cur] = {k: 0 for k in KEYS}
            funcs[cur]["instructions"] = 0
            continue
        if cur is None:
            continue
        m = re.match(r"\s*/\*[0-9a-f]+\*/\s+(?:@!?U?P\w+\s+)?([A-Z0-9_]+)", line)
        if not m:
            continue
        op = m.group(1)
        funcs[cur]["instructions"] += 1
        for k in KEYS:
            if op == k or op.startswith(k + "."):
                funcs[cur][k] += 1
    names = list(funcs)
    pretty = demangle(names)
    res = {}
    for raw, nice in zip(names, pretty):
        short = re.sub(r"\(.*", "", nice.replace("(anonymous namespace)::", "")).split("::")[-1]
        tag = short if short not in res else f"{short}#{raw[-12:]}"
        res[tag] = {k: v for k, v in funcs[raw].items() if v}
    doc = {"library": os.path.relpath(LIB, ROOT), "tool": "cuobjdump -sass (CUDA 12.9), counts per kernel",
           "legend": {"UTCIMMA": "tcgen05.mma kind::i8", "UTCHMMA": "tcgen05.mma kind::tf32/f16",
                      "UTMALDG": "TMA tensor load (cp.async.bulk.tensor)", "UBLKCP": "cp.async.bulk (1-D bulk copy)",
                      "LDTM": "tcgen05.ld (TMEM -> registers)", "STTM": "tcgen05.st", "UTCBAR": "tcgen05.commit",
                      "R2UR": "register -> uniform register moves"},
           "kernels": res}
    txt = json.dumps(doc, indent=1)
    if OUT:
        with open(OUT, "w") as f:
            f.write(txt + "\n")
    print(txt)


if __name__ == "__main__":
    main()
