"""Top shared-memory wavefront consumers of one kernel (ncu source page):
python tools/ncu_wave.py rep <kernel substring> <units> [top]"""
import sys

sys.path.insert(0, __file__.rsplit("/", 1)[0])
from ncu_sass import load  # noqa: E402


def main(rep, kre, units, top=30):
    hdr, data = load(rep, kre)
    I = hdr.index("Instructions Executed")
    W = hdr.index("L1 Wavefronts Shared")
    X = hdr.index("L1 Wavefronts Shared Excessive")
    Id = hdr.index("L1 Wavefronts Shared Ideal")
    f = lambda r, i: float(r[i]) if r[i] not in ("", "-") else 0.0
    tot = sum(f(r, W) for r in data)
    totx = sum(f(r, X) for r in data)
    print(f"wavefronts {tot:.3g} ({tot / units:.0f}/unit), excessive {totx:.3g} ({100 * totx / tot:.0f}%)")
    for r in sorted(data, key=lambda r: -f(r, X))[:top]:
        print(r[0][-5:], f"{f(r, I):9.0f} wf {f(r, W):9.0f} ideal {f(r, Id):9.0f}", r[1][:64])


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], float(sys.argv[3]), int(sys.argv[4]) if len(sys.argv) > 4 else 30)
