"""SASS opcode census of the hot kernels (cuobjdump -sass of the sm_100a objects).

For each kernel: the opcode histogram of the whole function and of its
hottest loop -- the backward branch whose body holds the most MUFU.EX2 (the
per-pair exponentials) -- with the per-pair FP32 issue count that the
roofline assumes: packed FFMA2 / FMUL2 / FADD2 count as two
FP32 lane operations per issue.

  python tools/sass_census.py > profiles/r02_sass_census.json
"""
import json
import os
import re
import subprocess
import sys
from collections import Counter

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OBJ = os.path.join(ROOT, "build", "obj")

KERNELS = {
    "allpairs.o": [
        "_ZN3gsb15k_rhs_sym_f32x2ILi12ELi256ELi1ELi128ELi8EEEvPK6float4iiffffPS1_",  # headline >= 150k
        "_ZN3gsb15k_rhs_sym_f32x2ILi12ELi128ELi2ELi256ELi4EEEvPK6float4iiffffPS1_",  # 40k - 150k
        "_ZN3gsb11k_rhs_f32x2ILi12ELi128ELi2ELi8EEEvPK6float4iiiiffffPS1_",  # gather >= 500k (shards)
        "_ZN3gsb11k_rhs_f32x2ILi8ELi128ELi3ELi8EEEvPK6float4iiiiffffPS1_",   # gather < 500k targets
        "_ZN3gsb12k_hess_f32x2ILi4ELi128EEEvPK6float4S3_iiiifffffPS1_",      # adjoint
        "_ZN3gsb9k_rhs_f64ILi4ELi128EEEvPK7double4iiiidPS1_",                # FP64 RHS
    ],
    "bh.o": [],  # filled by pattern below
}
BH_PATTERNS = [r"k_bh_wsIfLi0ELb0ELb0E", r"k_bh_grpIfLi0E", r"k_bh_wsIfLi1ELb1ELb0E"]

LINE = re.compile(r"/\*([0-9a-f]{4,})\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)\s*([^;]*);")
FP32_LANES = {"FFMA": 1, "FMUL": 1, "FADD": 1, "FFMA2": 2, "FMUL2": 2, "FADD2": 2, "FMNMX": 1}


def functions(obj):
    out = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True, check=True).stdout
    funcs, name, body = {}, None, []
    for ln in out.splitlines():
        m = re.search(r"Function : (\S+)", ln)
        if m:
            if name:
                funcs[name] = body
            name, body = m.group(1), []
            continue
        m = LINE.search(ln)
        if m and name:
            body.append((int(m.group(1), 16), m.group(3), m.group(4)))
    if name:
        funcs[name] = body
    return funcs


def census(body, sym=False):
    whole = Counter(op for _, op, _ in body)
    # loops: BRA to a lower address
    best, best_mufu = None, -1
    for addr, op, args in body:
        if op.startswith("BRA"):
            m = re.search(r"0x([0-9a-f]+)", args)
            if m and int(m.group(1), 16) < addr:
                lo = int(m.group(1), 16)
                seg = [o for a, o, _ in body if lo <= a <= addr]
                mufu = sum(1 for o in seg if o.startswith("MUFU"))
                # symmetric kernels: the smallest loop that evaluates pairs
                # AND updates the shared j accumulators (the source-step loop)
                if sym:
                    if not mufu or "STS.64" not in seg:
                        continue
                    if best is None or len(seg) < len(best[2]):
                        best, best_mufu = (lo, addr, seg), mufu
                    continue
                if mufu > best_mufu:
                    best, best_mufu = (lo, addr, seg), mufu
    res = {"instructions": len(body), "whole_function": dict(whole.most_common(40))}
    if best:
        lo, hi, seg = best
        c = Counter(seg)
        mufu = sum(v for k, v in c.items() if k.startswith("MUFU"))
        fp32 = sum(FP32_LANES.get(k.split(".")[0], 0) * v for k, v in c.items())
        res["hot_loop"] = {"range": [hex(lo), hex(hi)], "instructions": len(seg),
                           "opcodes": dict(c.most_common()),
                           "mufu": mufu, "fp32_lane_ops": fp32,
                           "fp32_lane_ops_per_mufu": fp32 / mufu if mufu else None}
    return res


def main():
    report = {"how": "cuobjdump -sass build/obj/*.o (sm_100a); tools/sass_census.py"}
    for obj, names in KERNELS.items():
        funcs = functions(os.path.join(OBJ, obj))
        if obj == "bh.o":
            names = [n for n in funcs if any(re.search(p, n) for p in BH_PATTERNS)]
        for n in names:
            if n in funcs:
                report[n] = census(funcs[n], sym="sym" in n)
    json.dump(report, sys.stdout, indent=1)
    print()


if __name__ == "__main__":
    main()
