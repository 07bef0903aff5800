"""Per-role breakdown of an als_umma_kernel ncu capture: warp-instructions and warp-stall samples per role,
from the CUDA-source correlation (-lineinfo) of als_umma_kernels.cu (role = the '// ---- <role>' section a
line falls in; inlined helpers count for the section that calls them, als_solve.cuh for the epilogue).
    python scripts/ncu_roles.py REP"""
import csv
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
src = open(os.path.join(ROOT, "paper_1511_02433_b200/csrc/als_umma_kernels.cu")).read().splitlines()
sections = []
for i, l in enumerate(src, 1):
    m = re.search(r"// ---- (\w+)", l)
    if m:
        sections.append((i, m.group(1)))
end = next(i for i, l in enumerate(src, 1) if "tcgen05.dealloc" in l)


def role(path, line):
    if path.endswith("als_solve.cuh"):
        return "epilogue(solve)"
    if not path.endswith("als_umma_kernels.cu"):
        return "other"
    r = "helpers/prologue"
    for s, n in sections:
        if line >= s and line < end:
            r = n
    return r


out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
kern, path, line, hdr = -1, "", 0, None
acc = {}
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        path = r[1]
        continue
    if r[0] == "Function Name":
        if path.endswith("als_umma_kernels.cu") or kern < 0:
            pass
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None:
        continue
    if r[0]:
        line = int(r[0])
        continue
    if len(r) > 8 and r[2].startswith("0x"):
        ie, si = int(r[7]), int(r[4])
        k = role(path, line)
        a = acc.setdefault(k, [0, 0])
        a[0] += ie
        a[1] += si
tot = sum(v[1] for v in acc.values())
for k, (ie, si) in sorted(acc.items(), key=lambda x: -x[1][1]):
    print(f"  {k:18s} instr {ie / 1e6:8.0f}M  samples {si / max(tot, 1) * 100:5.1f}%")
