"""Pipeline timeline of the fused operator (diagnostic): run one product with KGP_TC_TRACE
set, then print per-block event times of CTA (0, 0) relative to the MMA warp's issue of
the block (clock64 cycles).

    KGP_TC_TRACE=/tmp/tr.bin python tools/tc_probe.py 65536 32 2 fast gaussian 8 1
    python tools/tc_trace.py /tmp/tr.bin

Events: 0 producer issue, 1 dist-MMA issue, 2 dist issued, 3 set sees distances,
4 set loaded distances, 5 set sees free A stage, 6 set A tile ready, 7 MMA warp sees A tile,
8 MMA warp issued, 9 drain sees accumulators (per segment)."""
import sys

import numpy as np

NAMES = ["prod", "d_iss", "d_done", "s_dful", "s_dld", "s_aemp", "s_afull", "m_afull", "m_iss", "drain"]


def main():
    raw = np.fromfile(sys.argv[1], dtype=np.uint64)
    launches = raw.reshape(-1, 10, 256)
    tr = launches[-1].astype(np.int64)  # last launch
    t0 = tr[0, 0]
    valid = tr[7] > 0
    nb = int(valid.sum())
    print(f"blocks traced: {nb}")
    m = tr[7]
    per = np.diff(m[valid])
    print(f"MMA-warp period per block: median {np.median(per[8:]):.0f} cycles, mean {per[8:].mean():.0f}")
    print("block " + " ".join(f"{n:>8s}" for n in NAMES[:9]) + "   (cycles relative to m_afull of the block)")
    for t in range(8, min(nb, 40)):
        row = [tr[e, t] - m[t] if tr[e, t] else 0 for e in range(9)]
        print(f"{t:5d} " + " ".join(f"{v:8d}" for v in row))
    # averaged relative offsets over steady state
    rel = np.array([[tr[e, t] - m[t] for t in range(16, min(nb, 200))] for e in range(9)])
    print("mean  " + " ".join(f"{v:8.0f}" for v in rel.mean(axis=1)))
    # useful spans
    s = range(16, min(nb, 200))
    ld = np.mean([tr[4, t] - tr[3, t] for t in s])
    st = np.mean([tr[6, t] - tr[5, t] for t in s])
    wa = np.mean([tr[5, t] - tr[4, t] for t in s])
    hop = np.mean([tr[7, t] - tr[6, t] for t in s])
    iss = np.mean([tr[8, t] - tr[7, t] for t in s])
    print(f"set: dist load {ld:.0f}, wait for A stage {wa:.0f}, transform+store {st:.0f}; "
          f"A ready -> MMA warp sees it {hop:.0f}; MMA issue {iss:.0f}")
    d = np.mean([tr[5, t] - tr[8, t - 2] for t in s])
    print(f"MMA issue of block t-2 -> set sees its stage free (MMA execution + commit): {d:.0f}")


if __name__ == "__main__":
    main()
