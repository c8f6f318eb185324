"""L1 data-pipe budget of one kernel from an ncu source page: shared
wavefronts and global tag requests per barrier-delimited phase and per
opcode.  python tools/ncu_l1.py rep <kernel substring> <units>"""
import sys
from collections import defaultdict

sys.path.insert(0, __file__.rsplit("/", 1)[0])
from ncu_sass import load  # noqa: E402


def main(rep, kre, units):
    hdr, data = load(rep, kre)
    f = lambda r, k: float(r[hdr.index(k)]) if r[hdr.index(k)] not in ("", "-") else 0.0
    phase, ph = 0, defaultdict(lambda: [0.0, 0.0, 0.0])
    ops = defaultdict(lambda: [0.0, 0.0, 0.0])
    for r in data:
        src = r[1]
        op = src.split()[1] if src.startswith("@") else src.split()[0]
        i, w, g = (f(r, "Instructions Executed"), f(r, "L1 Wavefronts Shared"),
                   f(r, "L1 Tag Requests Global"))
        for d in (ph[phase], ops[op]):
            d[0] += i
            d[1] += w
            d[2] += g
        if op.startswith("BAR") or op.startswith("SYNCS"):
            phase += 1
    print(f"{'phase':>6} {'instr/u':>9} {'smem wf/u':>10} {'gtag/u':>8}")
    for p, (i, w, g) in sorted(ph.items()):
        print(f"{p:6d} {i / units:9.1f} {w / units:10.1f} {g / units:8.1f}")
    tot = [sum(v[k] for v in ph.values()) / units for k in range(3)]
    print(f"{'total':>6} {tot[0]:9.1f} {tot[1]:10.1f} {tot[2]:8.1f}")
    print("by opcode (smem wavefronts + global tags per unit):")
    for op, (i, w, g) in sorted(ops.items(), key=lambda kv: -(kv[1][1] + kv[1][2]))[:16]:
        print(f"  {op:24s} instr {i / units:7.1f}  smem {w / units:7.1f}  gtag {g / units:7.1f}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], float(sys.argv[3]))
