"""Bank-conflict and address-linearity check of the paired line kernel's
exchange-buffer layouts (AoS double2 slots, padded: slot(p) = p + (p >> K)).

For every exchange of a configuration (LOGM, P) it lists, per candidate K, the
128-bit wavefronts per quarter-warp access on the write and the read side
(1.0 = conflict free) and whether slot(p0(j) + r*S) - slot(p0(j)) is the same
for every thread (so the access is base register + immediate).
"""
import sys

def log2(x): return x.bit_length() - 1

def paired_bfly(tl, q, B, T):
    NS = B * T
    if tl == 0: return q * T
    return tl + q * T if q < B // 2 else NS - tl - (q - B // 2) * T

def slot(p, K): return p + (p >> K) if K else p

def wavefronts(addr_lists):
    """addr_lists: per thread (ordered by tl) slot index of one access; 16-byte
    slots, 8 bank groups; quarter-warp phases of 8 lanes."""
    tot, n = 0, 0
    for i in range(0, len(addr_lists), 8):
        lanes = addr_lists[i:i + 8]
        cnt = {}
        for a in set(lanes):  # same address broadcasts
            cnt[a % 8] = cnt.get(a % 8, 0) + 1
        tot += max(cnt.values())
        n += 1
    return tot / n

def check(LOGM, P, verbose=True):
    M = 1 << LOGM; T = M // P; LP = log2(P)
    SPLIT = LOGM % LP == 0
    REM = 1 if SPLIT else LOGM % LP
    R0 = 1 << REM; B0 = P // R0; NS0 = M // R0
    # exchanges: (name, write (NSL, R, paired), read (R, paired))
    ex = []
    nsl = 0
    while True:  # forward
        R = P // 2 if (SPLIT and LOGM - nsl == LP) else P
        nx = nsl + log2(R)
        last = (LOGM - nx) == REM
        if last:
            ex.append((f"fwd w(NS=2^{nsl},R={R}) r(paired R0={R0})", (nsl, R, False), (R0, True)))
            break
        RN = P // 2 if (SPLIT and LOGM - nx == LP) else P
        ex.append((f"fwd w(NS=2^{nsl},R={R}) r(R={RN})", (nsl, R, False), (RN, False)))
        nsl = nx
    nsl = REM  # inverse: paired stage at NSL=0 first
    RN = P // 2 if (SPLIT and nsl == REM) else P
    ex.append((f"inv w(paired NS=1,R0={R0}) r(R={RN})", (0, R0, True), (RN, False)))
    while True:
        R = P // 2 if (SPLIT and nsl == REM) else P
        nx = nsl + log2(R)
        if nx >= LOGM: break
        RN = P
        ex.append((f"inv w(NS=2^{nsl},R={R}) r(R={RN})", (nsl, R, False), (RN, False)))
        nsl = nx
    res = {}
    for name, (wn, wR, wp), (rR, rp) in ex:
        rows = []
        for K in (0, 3, 4, 5):
            # write side
            Bw = P // wR; NS = 1 << wn
            ww, lin = [], True
            for q in range(Bw):
                for r in range(wR):
                    addrs = []
                    for tl in range(T):
                        j = paired_bfly(tl, q, Bw, T) if wp else tl + q * T
                        base = ((j >> wn) << (wn + log2(wR))) + (j & (NS - 1))
                        addrs.append(slot(base + r * NS, K))
                        if slot(base + r * NS, K) - slot(base, K) != slot(r * NS, K): lin = False
                    ww.append(wavefronts(addrs))
            Br = P // rR
            rw = []
            for q in range(Br):
                for r in range(rR):
                    addrs = []
                    for tl in range(T):
                        j = paired_bfly(tl, q, Br, T) if rp else tl + q * T
                        addrs.append(slot(j + r * (M // rR), K))
                        if slot(j + r * (M // rR), K) - slot(j, K) != slot(r * (M // rR), K): lin = False
                    rw.append(wavefronts(addrs))
            rows.append((K, sum(ww) / len(ww), sum(rw) / len(rw), lin))
        res[name] = rows
        if verbose:
            print(f"  {name}")
            for K, w, r, lin in rows:
                print(f"     K={K}: write {w:.3f}  read {r:.3f}  linear={lin}")
    return res

if __name__ == "__main__":
    cfgs = [(11, 16), (10, 16), (12, 16), (13, 16)]
    for LOGM, P in cfgs:
        print(f"M=2^{LOGM} P={P}")
        check(LOGM, P)
