"""numpy model of the GPU block one-sided Jacobi (sweep counts of preconditioning/ordering variants on harvested theta matrices: python tools/jacobi_model.py Q1,Q2 VARIANT with M_<q>.npy files from a cfg3 steady state)."""
import numpy as np, sys, time
EPS = 1.1102230246251565e-16

def tourney(N, rho, p):
    if p == 0: a, b = rho, N - 1
    else: a, b = (rho + p) % (N - 1), (rho - p + N - 1) % (N - 1)
    return min(a, b), max(a, b)

def rotations(G, I, Jc, tol, noise2, fro):
    a = G[I, I].real; b = G[Jc, Jc].real; g = G[I, Jc]
    lo = np.minimum(a, b); hi = np.maximum(a, b)
    g2 = np.abs(g) ** 2
    act = (hi > noise2) & (lo > 1e-250 * hi) & (g2 > (tol * fro) ** 2 * lo)
    delta = b - a
    rho2 = delta ** 2 + 4 * g2
    with np.errstate(all='ignore'):
        rr = 1 / np.sqrt(rho2)
        c2 = 0.5 + 0.5 * np.abs(delta) * rr
        c = np.sqrt(c2)
        s = np.abs(g) * rr / c
        s = np.where(delta < 0, -s, s)
        e = g / np.abs(g)
    c = np.where(act, c, 1.0); s = np.where(act, s, 0.0); e = np.where(act, e, 1.0)
    return act, c, s, e

def inner(G, pairs_fn, nrounds, tol, noise2, fro, W2, max_inner=1):
    Q = np.eye(W2, dtype=complex)
    first = 0
    for it in range(max_inner):
        any_ = 0
        for rho in range(nrounds):
            I, Jc = pairs_fn(rho)
            act, c, s, e = rotations(G, I, Jc, tol, noise2, fro)
            n = int(act.sum()); any_ += n
            if n == 0: continue
            J = np.eye(W2, dtype=complex)
            J[I, I] = c; J[I, Jc] = s; J[Jc, I] = -s * np.conj(e); J[Jc, Jc] = c * np.conj(e)
            G = J.conj().T @ G @ J
            Q = Q @ J
        if it == 0: first = any_
        if any_ == 0: break
    return first, Q

def jacobi(Z, w=16, full_every=False, max_inner=1, tol_factor=4.0, max_sweeps=40):
    r, c = Z.shape
    Z = Z.copy()
    nb = (c + w - 1) // w; nb += nb & 1
    fro = np.linalg.norm(Z); noise2 = (1e-14 * fro) ** 2
    tol = tol_factor * np.sqrt(r) * EPS
    W2 = 2 * w
    full_pairs = [np.array([tourney(W2, rho, p) for p in range(w)]) for rho in range(W2 - 1)]
    fp = lambda rho: (full_pairs[rho][:, 0], full_pairs[rho][:, 1])
    cp = lambda rho: (np.arange(w), w + (np.arange(w) + rho) % w)
    for sweep in range(max_sweeps):
        dirty = False
        for rho in range(nb - 1):
            for v in range(nb // 2):
                I, J = tourney(nb, rho, v)
                cols = np.r_[I * w:(I + 1) * w, J * w:(J + 1) * w]
                P = Z[:, cols]
                G = P.conj().T @ P
                full = full_every or rho == 0
                nrot, Q = inner(G, fp if full else cp, W2 - 1 if full else w, tol, noise2, fro, W2, max_inner)
                if nrot:
                    dirty = True
                    Z[:, cols] = P @ Q
        if not dirty:
            return sweep, Z
    return max_sweeps, Z

def precond(M, double=True):
    R1 = np.linalg.qr(M, mode='r')
    Y = R1.conj().T
    if not double: return Y
    R2 = np.linalg.qr(Y, mode='r')
    return R2.conj().T

def precond_n(M, n, pivot=True):
    """n alternating QRs (R^H of the previous factor), first with static column pivoting."""
    if pivot:
        M = M[:, np.argsort(-np.linalg.norm(M, axis=0))]
    Y = M
    for _ in range(n):
        Y = np.linalg.qr(Y, mode='r').conj().T
    return Y

if __name__ == "__main__":
    qs = [int(x) for x in sys.argv[1].split(',')]
    variant = sys.argv[2]
    for q in qs:
        M = np.load(f'M_{q}.npy')
        kw = {}
        dbl = True
        if variant == 'full': kw['full_every'] = True
        if variant == 'inner2': kw['max_inner'] = 2
        if variant == 'inner3': kw['max_inner'] = 3
        if variant == 'w32': kw['w'] = 32
        if variant == 'w8': kw['w'] = 8
        if variant == 'single': dbl = False
        Z = precond(M, dbl)
        if variant.startswith('qr'):
            Z = precond_n(M, int(variant[2:]))
        if variant == 'sort':
            Z = Z[:, np.argsort(-np.linalg.norm(Z, axis=0))]
        t = time.time()
        sw, Zf = jacobi(Z, **kw)
        s = np.sort(np.linalg.norm(Zf, axis=0))[::-1]
        sref = np.linalg.svd(M, compute_uv=False)
        print(variant, q, 'sweeps', sw, 'maxrel', np.max(np.abs(s - sref)) / sref[0], '%.1fs' % (time.time() - t), flush=True)
