"""Rebuild Python model objects from the golden fixtures (tests/golden/*.npz)."""
from __future__ import annotations

import numpy as np

from paper_2105_04150_b200.types import (BoundaryConditions, Corrections, DamageLaw, DamageModel,
                                         ModelBundle, NeighborList, ParticleSet, RampKind,
                                         RampProfile, SimulationState, make_state)


def random_case(d, seed):
    pre = f"s{seed}_"
    law = d[pre + "law"]
    nbp = int(law[1])
    dl = DamageLaw(float(law[0]), list(law[2:2 + nbp]), list(law[2 + nbp:2 + 2 * nbp]))
    n = d[pre + "volume"].size
    p = ParticleSet(d[pre + "coords"].copy(), d[pre + "volume"].copy(), d[pre + "density"].copy(),
                    np.zeros(n, np.uint16))
    fam = NeighborList(d[pre + "entries"].copy(), d[pre + "n_neigh"].copy(),
                       d[pre + "initial"].copy(), int(d[pre + "group"]), 0.0, None)
    st = SimulationState(d[pre + "u"].copy(), np.zeros(3 * n), np.zeros(3 * n), 0, fam,
                         d[pre + "history"].copy())
    corr = Corrections(d[pre + "lambda"].copy() if pre + "lambda" in d else None,
                       d[pre + "beta"].copy() if pre + "beta" in d else None, None)
    return p, DamageModel([dl]), corr, st


def sim_case(d, name):
    pre = name + "_"
    n = d[pre + "volume"].size
    p = ParticleSet(d[pre + "coords"].copy(), d[pre + "volume"].copy(), d[pre + "density"].copy(),
                    np.zeros(n, np.uint16))
    laws = []
    for c, bp, f, k in zip(d[pre + "law_c"], d[pre + "law_bp"], d[pre + "law_f"], d[pre + "law_n"]):
        laws.append(DamageLaw(float(c), list(bp[:k]), list(f[:k])))
    model = DamageModel(laws, float(d[pre + "damping"]))
    corr = Corrections(d[pre + "lambda"].copy() if pre + "lambda" in d else None,
                       d[pre + "beta"].copy() if pre + "beta" in d else None, None)
    ramps = [RampProfile(RampKind(int(r[0])), int(r[1]), float(r[2])) for r in d[pre + "ramps"]]
    names = list(d[pre + "tip_names"])
    offs = d[pre + "tip_offsets"]
    nodes = d[pre + "tip_nodes"]
    tips = {str(nm): [int(x) for x in nodes[offs[k]:offs[k + 1]]] for k, nm in enumerate(names)}
    bc = BoundaryConditions(d[pre + "bc_kind"].copy(), d[pre + "bc_mag"].copy(),
                            d[pre + "bc_ramp"].copy(), ramps, d[pre + "bc_nofail"].copy(), tips)
    fam = NeighborList(d[pre + "entries"].copy(), d[pre + "n_neigh"].copy(),
                       d[pre + "initial"].copy(), int(d[pre + "group"]), float(d[pre + "horizon"]),
                       d[pre + "bond_type"].copy() if pre + "bond_type" in d else None)
    bundle = ModelBundle(p, model, corr, bc, float(d[pre + "dt"]))
    state = make_state(fam, model.needs_history())
    if pre + "u0" in d:
        state.u = d[pre + "u0"].copy()
    steps, write_every, first, integrator = (int(x) for x in d[pre + "opts"])
    return bundle, state, steps, write_every, first, integrator


def tips_table(result):
    rows = []
    for name in sorted(result.tips):
        for r in result.tips[name]:
            rows.append([r.step, *r.mean_u, *r.mean_v, *r.mean_a, *r.body_force_sum,
                         *r.external_force_sum])
    return np.array(rows) if rows else np.zeros((0, 16))


def bits(a):
    return np.ascontiguousarray(a).view(np.uint8)


def same_bits(a, b) -> bool:
    a = np.ascontiguousarray(a)
    b = np.ascontiguousarray(b)
    return a.shape == b.shape and a.dtype == b.dtype and np.array_equal(bits(a), bits(b))
