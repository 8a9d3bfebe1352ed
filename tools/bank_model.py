"""Shared-memory bank model of the Stockham exchanges in the column layout (8-byte
elements, 16 slots per wavefront): worst wavefronts per warp instruction for
the writes and reads of every pass, plain vs padded layouts (PadColLayout)."""
import itertools
def sched(L, P):
    K = L.bit_length()-1; KP = P.bit_length()-1
    R0 = (1 << (K % KP)) if K % KP else P
    npass = 1 + K//KP if K % KP else K//KP
    passes=[]
    for p in range(npass):
        R = R0 if p == 0 else P
        Ns = 1 if p == 0 else R0 * (1 << (KP*(p-1)))
        passes.append((R, Ns))
    return passes
def wavefronts(addrs):
    slots={}
    for a in addrs: slots.setdefault(a % 16, set()).add(a)
    return max(len(v) for v in slots.values())
def analyze(L, P, COLS, layout):
    T = L // P
    NTC = COLS*T
    res=[]
    for pi,(R,Ns) in enumerate(sched(L,P)):
        NB = P // R
        worst_w=0; worst_r=0
        for w in range(NTC//32):
            lanes=[w*32+l for l in range(32)]
            # writes (except last pass)
            if pi < len(sched(L,P))-1:
                for m in range(NB):
                    for q in range(R):
                        addrs=[]
                        for tid in lanes:
                            c = tid % COLS; t = tid // COLS
                            j = t + m*T
                            e = (j//Ns)*Ns*R + (j % Ns) + q*Ns
                            addrs.append(layout(e,c))
                        worst_w=max(worst_w,wavefronts(addrs))
                # reads after exchange
                for s_ in range(P):
                    addrs=[layout((tid//COLS)+s_*T, tid%COLS) for tid in lanes]
                    worst_r=max(worst_r,wavefronts(addrs))
        res.append((pi,R,Ns,worst_w,worst_r))
    return res
for COLS in (4, 8, 16):
    for name, lay in (("plain", lambda e,c,C=COLS: e*C+c), ("pad16", lambda e,c,C=COLS: e*C + c + C*(e>>4)), ("pad8", lambda e,c,C=COLS: e*C + c + C*(e>>3)), ("pad16+1", lambda e,c,C=COLS: e*C + c + (e>>4))):
        print(COLS, name, analyze(2048, 16, COLS, lay))
print("---- PP=32")
for L in (256, 512, 1024):
  for COLS in (8, 16):
    for name, lay in (("plain", lambda e,c,C=COLS: e*C+c), ("pad16", lambda e,c,C=COLS: e*C + c + C*(e>>4))):
        print(L, COLS, name, analyze(L, 32, COLS, lay))
print("---- pad by first radix")
for P in (16, 32):
  for L in (64, 128, 256, 512, 1024, 2048):
    if P == 32 and L > 1024: continue
    R0 = sched(L, P)[0][0]; sh = R0.bit_length()-1
    for COLS in (4, 8, 16, 32):
        if COLS * (L // P) % 32: continue
        lay = lambda e,c,C=COLS,sh=sh: e*C + c + C*(e>>sh)
        r = analyze(L, P, COLS, lay)
        rp = analyze(L, P, COLS, lambda e,c,C=COLS: e*C+c)
        print(P, L, COLS, "R0", R0, "padded", [(x[3],x[4]) for x in r], "plain", [(x[3],x[4]) for x in rp])
