"""SASS listing of one kernel from an ncu report with executed-instruction
counts and stall samples: python tools/ncu_sass.py rep <kernel substring> [top]"""
import csv
import subprocess
import sys
from collections import Counter


def load(rep, kre):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    names = [i for i, r in enumerate(rows) if r and r[0] == "Kernel Name"]
    k = [i for i in names if kre in rows[i][1]][0]
    nxt = [i for i in names if i > k]
    hdr = rows[k + 1]
    return hdr, rows[k + 2:(nxt[0] if nxt else None)]


def main(rep, kre, top=40):
    hdr, data = load(rep, kre)
    I, S = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
    f = lambda r, i: float(r[i]) if r[i] not in ("", "-") else 0.0
    ops = Counter()
    for r in data:
        ops[r[1].split()[0] if not r[1].startswith("@") else r[1].split()[1]] += f(r, I)
    tot = sum(ops.values())
    print("opcode mix:", ", ".join(f"{o} {100 * c / tot:.1f}%" for o, c in ops.most_common(18)))
    mode = sys.argv[4] if len(sys.argv) > 4 else "list"
    if mode == "list":
        for r in data:
            print(f"{r[0][-5:]} {f(r, I):>9.0f} {f(r, S):>6.0f}  {r[1][:90]}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 40)
