"""Collects per-CTA sweep times (pmf_ctx_debug_sweep_profile) and layout features under several CTA
partition cost models (PMF_UNIT_COST) so the cost model can be fitted by regression offline:

    python scripts/cta_fit.py collect gpurun_out/cta_data.npz      # on the GPU box
    python scripts/cta_fit.py fit gpurun_out/cta_data.npz          # here

Different cost models give different per-CTA mixes of long / medium / short units, which breaks the
collinearity a single balanced layout has (every CTA has the same modelled cost)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

# PMF_UNIT_COST: step_a x3, per_step_a x3, step_b x3, per_step_b x3, per_entry x3, per_unit x3,
# per_piece (ps); "" = the library default
MODELS = ["", "1,1,1,0,0,0,1,1,1,0,0,0,1000,1000,1000,64000,64000,64000,0",
          "1,1,1,0,0,0,1,1,1,0,0,0,1000,1000,1000,0,0,0,0",
          "64,32,16,2835,3912,0,1,1,1,0,0,0,66,0,168,2653,0,0,0",
          "64,32,16,2835,3912,0,1,1,1,0,0,0,66,0,168,2653,0,0,14000000"]


def collect(out):
    import bench
    import paper_1511_02433_b200 as P
    m0, n0 = bench.CONFIGS["netflix-ccdpp"][:2]
    train, probe = bench.make_data("netflix-ccdpp")
    A = P.RatingsMatrix.from_triplets(train, m0, n0)
    data = {}
    for mi, m in enumerate(MODELS):
        if m:
            os.environ["PMF_UNIT_COST"] = m
        else:
            os.environ.pop("PMF_UNIT_COST", None)
        ctx = P.Context(A)
        ctx.ccdpp_begin(P.CcdConfig(k=40, lam=0.05, outer_iters=1, inner_iters=15, seed=1))
        ctx.ccdpp_iterate(1)
        for side in (0, 1):
            for promote in (0, 1):
                durs = []
                for _ in range(3):
                    clk, st = ctx.debug_sweep_profile(side, bool(promote))
                    durs.append((clk[:, 1] - clk[:, 0]) / 1e3)
                d = np.median(np.array(durs), axis=0)
                data[f"m{mi}_s{side}_p{promote}_dur"] = d
                data[f"m{mi}_s{side}_p{promote}_st"] = st
                print(f"model {m} side {side} promote {promote}: max {d.max():.1f} avg {d.mean():.1f} "
                      f"min {d.min():.1f} us", file=sys.stderr)
        ctx.close()
        del ctx
    np.savez(out, **data)


# kernel variants: lanes-per-group 8/4/2 with unroll (UA, UB, UC); plain CSC = V2, promote = V0
UNROLL = {"plain": (2, 2, 2), "promote": (8, 4, 4), "plain_csr": (4, 2, 2)}


def features(st, unroll):
    cols = []
    for c in range(3):
        j = {1: 0, 2: 1, 4: 2, 8: 3}[unroll[c]]
        cols.append(st[:, 9 + 3 * j + c])       # group-steps of class c
    for c in range(3):
        cols.append(st[:, 6 + c])               # entries of class c
    for c in range(3):
        cols.append(st[:, c])                   # units of class c
    cols.append(st[:, 4])                       # pieces
    return np.column_stack(cols).astype(float)


NAMES = ["steps_L", "steps_M", "steps_S", "ent_L", "ent_M", "ent_S", "units_L", "units_M", "units_S", "pieces"]


def fit(path):
    z = np.load(path)
    nm = len([k for k in z.files if k.endswith("_s0_p0_dur")])
    for side in (0, 1):
        for promote in (0, 1):
            un = UNROLL["promote"] if promote else (UNROLL["plain_csr"] if side == 0 else UNROLL["plain"])
            X = np.concatenate([features(z[f"m{m}_s{side}_p{promote}_st"], un) for m in range(nm)])
            d = np.concatenate([z[f"m{m}_s{side}_p{promote}_dur"] for m in range(nm)])
            for sel, label in ((slice(None), "all"), ):
                Xs = np.column_stack([X[sel], np.ones(len(d))])
                # non-negative least squares by active-set pruning
                active = list(range(Xs.shape[1]))
                while True:
                    coef, *_ = np.linalg.lstsq(Xs[:, active], d, rcond=None)
                    neg = [a for a, c in zip(active, coef) if c < 0 and a != Xs.shape[1] - 1]
                    if not neg:
                        break
                    active.remove(neg[0])
                full = np.zeros(Xs.shape[1])
                full[active] = coef
                pred = Xs @ full
                print(f"side {side} promote {promote}: rms {np.sqrt(np.mean((pred - d) ** 2)):.2f} us "
                      f"(dur range {d.min():.0f}-{d.max():.0f})")
                print("   " + "  ".join(f"{n}={c * 1e3:.3f}ns" for n, c in zip(NAMES + ["const"], full) if c)
                      + f"  const={full[-1]:.1f}us")
            for m in range(nm):
                dd = z[f"m{m}_s{side}_p{promote}_dur"]
                print(f"     model {MODELS[m]:>20s}: max {dd.max():6.1f} avg {dd.mean():6.1f} min {dd.min():6.1f}")


def fit_step(path, side=1, inner=15):
    """Cost model for the time of a whole rank-one step on one side: (inner - 1) plain sweeps + 1 promote
    per CTA, as per_entry[c] * entries + per_unit[c] * units (+ per_piece * pieces), non-negative least
    squares over every collected partition.  Prints the PMF_UNIT_COST string (no step terms)."""
    z = np.load(path)
    nm = len([k for k in z.files if k.endswith("_s0_p0_dur")])
    X, d = [], []
    for m in range(nm):
        st = z[f"m{m}_s{side}_p0_st"]
        y = (inner - 1) * z[f"m{m}_s{side}_p0_dur"] + z[f"m{m}_s{side}_p1_dur"]
        X.append(np.column_stack([st[:, 6], st[:, 7], st[:, 8], st[:, 0], st[:, 1], st[:, 2], st[:, 4]]).astype(float))
        d.append(y)
    X, d = np.concatenate(X), np.concatenate(d)
    Xs = np.column_stack([X, np.ones(len(d))])
    active = list(range(Xs.shape[1]))
    while True:
        coef, *_ = np.linalg.lstsq(Xs[:, active], d, rcond=None)
        neg = [a for a, c in zip(active, coef) if c < 0 and a != Xs.shape[1] - 1]
        if not neg:
            break
        active.remove(neg[0])
    full = np.zeros(Xs.shape[1])
    full[active] = coef
    pred = Xs @ full
    print(f"side {side} step ({inner - 1} plain + 1 promote): rms {np.sqrt(np.mean((pred - d) ** 2)):.1f} us "
          f"(range {d.min():.0f}-{d.max():.0f})")
    names = ["ent_L", "ent_M", "ent_S", "units_L", "units_M", "units_S", "pieces", "const"]
    print("   " + "  ".join(f"{n}={c * 1e3:.3f}ns" for n, c in zip(names, full)))
    ps = lambda x: int(round(x * 1e6))  # us -> the model's integer units (ps)
    cost = [1, 1, 1, 0, 0, 0, 1, 1, 1, 0, 0, 0, ps(full[0]), ps(full[1]), ps(full[2]), ps(full[3]), ps(full[4]),
            ps(full[5]), ps(full[6])]
    print("PMF_UNIT_COST=" + ",".join(str(c) for c in cost))


if __name__ == "__main__":
    if sys.argv[1] == "collect":
        collect(sys.argv[2])
    elif sys.argv[1] == "fit_step":
        fit_step(sys.argv[2])
    else:
        fit(sys.argv[2])
