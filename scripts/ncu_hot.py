"""Per-kernel hot SASS instructions from an ncu report (warp stall samples): python scripts/ncu_hot.py REP [N]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(out.splitlines()))
blocks, cur, hdr = [], None, None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = []
        blocks.append((r[1][:80], cur))
        continue
    if r and r[0] == "Address":
        hdr = r
        continue
    if cur is not None and len(r) > 5:
        cur.append(r)
si = hdr.index("Warp Stall Sampling (All Samples)")
ie = hdr.index("Instructions Executed")
for name, b in blocks:
    tot = sum(int(x[si]) for x in b)
    print(f"== {name}  samples {tot}  warp-instr {sum(int(x[ie]) for x in b)}")
    top = sorted(range(len(b)), key=lambda i: -int(b[i][si]))[:n]
    for i in sorted(top):
        print(f"{i:6d} {int(b[i][si]) / tot * 100:5.1f}% {b[i][ie]:>10s}  {b[i][1][:90]}")

if len(sys.argv) > 3:  # region breakdown: markers -> index of first occurrence
    for name, b in blocks[:1]:
        tot = sum(int(x[si]) for x in b)
        marks = [(i, x[1].strip()[:60]) for i, x in enumerate(b) if any(
            m in x[1] for m in ("UTMALDG", "UTCHMMA", "LDTM", "LDGSTS", "SYNCS.ARRIVE", "BAR.SYNC", "EXIT", "MUFU.SQRT", "MUFU.RSQ"))]
        for i, t in marks:
            print(f"   mark {i:6d} {t}")
        step = int(sys.argv[3])
        for a in range(0, len(b), step):
            sub = sum(int(x[si]) for x in b[a:a + step])
            if sub / tot > 0.003:
                print(f"   [{a:6d},{a + step:6d}) {sub / tot * 100:5.1f}%")
