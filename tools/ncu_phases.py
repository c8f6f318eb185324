"""Per-phase (barrier-delimited) instruction and stall split of one kernel
from an ncu report: python tools/ncu_phases.py rep.ncu-rep <kernel regex> <units>"""
import csv
import subprocess
import sys


def main(rep, kre, units):
    """kre: substring of the demangled kernel name (first matching launch)."""
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    names = [i for i, r in enumerate(rows) if r and r[0] == "Kernel Name"]
    k = [i for i in names if kre in rows[i][1]][0]
    nxt = [i for i in names if i > k]
    hi = k + 1
    hdr = rows[hi]
    data = rows[hi + 1:(nxt[0] if nxt else None)]
    I = hdr.index("Instructions Executed")
    S = hdr.index("Warp Stall Sampling (All Samples)")

    def f(r, i):
        try:
            return float(r[i])
        except ValueError:
            return 0.0
    phase, acc, st, first = 0, {}, {}, {}
    for r in data:
        acc[phase] = acc.get(phase, 0) + f(r, I)
        st[phase] = st.get(phase, 0) + f(r, S)
        first.setdefault(phase, r[0][-5:])
        if "BAR.SYNC" in r[1] or "BAR.RED" in r[1]:
            phase += 1
    tot, tots = sum(acc.values()), sum(st.values())
    print(f"{kre}: {tot:.3g} warp-instr, {tot / units:.0f} per unit")
    for p in acc:
        print(f"  phase {p} @{first[p]}: instr {100 * acc[p] / tot:5.1f}%  stall "
              f"{100 * st[p] / tots:5.1f}%  ({acc[p] / units:.0f} per unit)")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], float(sys.argv[3]))
