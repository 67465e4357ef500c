"""Generate the golden vectors by running the REFERENCE package itself.

Run in the dev container, where the reference is importable:

    python tests/golden/make_golden.py            # imports /root/reference/pkg/src

Outputs (committed): vote_c7.npz, vote_grid.npz, verify_greedy.npz,
verify_stoch.npz, verify_stoch_bigv.json, weights_trace.json, selector_trace.json.
Nothing on the GPU box or in the product imports the reference; tests read
only these files.
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF = os.environ.get("AGGSPEC_REF_SRC", "/root/reference/pkg/src")
sys.path.insert(0, REF)

from aggspec.core import EngineConfig, ProbDist, seeded_rng  # noqa: E402
from aggspec.selector import MonitorSample, SelectorState, maybe_adjust, observe  # noqa: E402
from aggspec.verification import verify  # noqa: E402
from aggspec.voting import WeightTable, merge, record_acr, select_majority, update_weights  # noqa: E402


class CountingRng:
    """Proxy recording every uniform the reference draws (verify only calls .random())."""

    def __init__(self, rng):
        self.rng = rng
        self.draws: list[float] = []

    def random(self):
        u = self.rng.random()
        self.draws.append(u)
        return u


def pad(arr_list, shape, fill=-1, dtype=np.int32):
    out = np.full(shape, fill, dtype)
    for i, a in enumerate(arr_list):
        a = np.asarray(a)
        out[(i,) + tuple(slice(0, d) for d in a.shape)] = a
    return out


def gen_vote_c7():
    """tests/test_acceptance.py:288-313 instances (default_rng(42)) + the Fig.-5 instance."""
    gen = np.random.default_rng(42)
    toks, ws, Ks, Ss, paths, voted = [], [], [], [], [], []
    inst = [([[0, 1, 3], [0, 1, 4], [0, 2, 5]], [0.5, 0.4, 0.6], [1, 2, 3])]
    for _ in range(1000):
        n = int(gen.integers(1, 5))
        s = int(gen.integers(1, 5))
        d = [[int(t) for t in gen.integers(0, 5, size=s)] for _ in range(n)]
        w = [float(gen.uniform(0.1, 5.0)) for _ in range(n)]
        inst.append((d, w, list(range(n))))
    for d, w, ids in inst:
        out = select_majority(merge(list(zip(ids, d)), dict(zip(ids, w))))
        toks.append(d)
        ws.append(w)
        Ks.append(len(d))
        Ss.append(len(d[0]))
        paths.append(out.tokens)
        voted.append(ids.index(out.voted_ssm))
    N = len(inst)
    np.savez_compressed(
        os.path.join(HERE, "vote_c7.npz"),
        tokens=pad(toks, (N, 4, 4)), weights=pad(ws, (N, 4), 0.0, np.float64),
        K=np.array(Ks, np.int32), S=np.array(Ss, np.int32),
        path=pad(paths, (N, 4)), voted=np.array(voted, np.int32),
    )


def reachable_weight(gen):
    a, b = int(gen.integers(0, 40)), int(gen.integers(0, 40))
    w = 1.0
    seq = ["r"] * a + ["p"] * b
    gen.shuffle(seq)
    for op in seq:  # the exact fp64 op sequence update_weights applies
        w = min(max(w * (1.25 if op == "r" else 0.8), 1e-3), 1e3)
    return w


def gen_vote_grid(n_inst=10000):
    """cfg4 extents: K 1-8, S 1-16, small token alphabets to force collisions,
    weights reachable via x1.25/x0.8 (half) or U(0.1, 5) (half); 20% of the
    instances use shuffled non-contiguous ids so draft order != id order."""
    gen = np.random.default_rng(20240226)
    toks, ws, Ks, Ss, paths, voted, ranks = [], [], [], [], [], [], []
    for i in range(n_inst):
        K = int(gen.integers(1, 9))
        S = int(gen.integers(1, 17))
        alpha = int(gen.choice([2, 3, 5, 8, 50000]))
        d = gen.integers(0, alpha, size=(K, S))
        # make drafts share prefixes often
        for k in range(1, K):
            if gen.random() < 0.5:
                src = int(gen.integers(0, k))
                cut = int(gen.integers(0, S + 1))
                d[k, :cut] = d[src, :cut]
        if i % 2 == 0:
            w = [reachable_weight(gen) for _ in range(K)]
        else:
            w = [float(gen.uniform(0.1, 5.0)) for _ in range(K)]
        if i % 5 == 0:
            ids = [int(x) for x in gen.permutation(100)[:K]]
        else:
            ids = list(range(K))
        drafts = [(ids[k], [int(t) for t in d[k]]) for k in range(K)]
        out = select_majority(merge(drafts, dict(zip(ids, w))))
        order = sorted(range(K), key=lambda k: ids[k])
        rank = [0] * K
        for r, k in enumerate(order):
            rank[k] = r
        toks.append(d)
        ws.append(w)
        Ks.append(K)
        Ss.append(S)
        paths.append(out.tokens)
        voted.append(ids.index(out.voted_ssm))
        ranks.append(rank)
    N = n_inst
    np.savez_compressed(
        os.path.join(HERE, "vote_grid.npz"),
        tokens=pad(toks, (N, 8, 16)), weights=pad(ws, (N, 8), 0.0, np.float64),
        rank=pad(ranks, (N, 8)), K=np.array(Ks, np.int32), S=np.array(Ss, np.int32),
        path=pad(paths, (N, 16)), voted=np.array(voted, np.int32),
    )


def gen_verify_greedy(n=5000, V=50):
    """verify() on point masses: records accepted, emitted
    and the number of uniforms consumed."""
    gen = np.random.default_rng(7)
    drafts, tgts, accs, ems, nds, Ss = [], [], [], [], [], []
    for i in range(n):
        s = int(gen.integers(1, 17))
        p_agree = float(gen.choice([0.0, 0.5, 0.8, 0.95, 1.0]))
        tgt = gen.integers(0, V, size=s + 1)
        dr = np.where(gen.random(s) < p_agree, tgt[:s], gen.integers(0, V, size=s))
        rng = CountingRng(seeded_rng(i, f"verify/req-{i:03d}"))
        res = verify([int(t) for t in dr], [ProbDist.point_mass(int(t), V) for t in dr],
                     [ProbDist.point_mass(int(t), V) for t in tgt], rng)
        drafts.append(dr)
        tgts.append(tgt)
        accs.append(res.accepted_count)
        ems.append(res.emitted)
        nds.append(len(rng.draws))
        Ss.append(s)
    np.savez_compressed(
        os.path.join(HERE, "verify_greedy.npz"),
        draft=pad(drafts, (n, 16)), target_argmax=pad(tgts, (n, 17)),
        S=np.array(Ss, np.int32), accepted=np.array(accs, np.int32),
        emitted=pad(ems, (n, 17)), n_draws=np.array(nds, np.int32),
    )


def gen_verify_stoch():
    """Full stochastic verify() with Dirichlet q/o; records the uniforms drawn."""
    gen = np.random.default_rng(11)
    groups = {}
    for V, n, smax in ((5, 1500, 6), (37, 400, 6), (300, 60, 4)):
        qs, os_, drafts, us, accs, ems, Ss = [], [], [], [], [], [], []
        for i in range(n):
            s = int(gen.integers(1, smax + 1))
            conc = float(gen.choice([0.1, 1.0, 5.0]))
            q = [ProbDist(gen.dirichlet(np.full(V, conc))) for _ in range(s)]
            o = [ProbDist(gen.dirichlet(np.full(V, conc))) for _ in range(s + 1)]
            if gen.random() < 0.2:  # identical models on some positions
                for j in range(s):
                    if gen.random() < 0.5:
                        o[j] = q[j]
            dr = [q[j].sample(gen) for j in range(s)]
            rng = CountingRng(seeded_rng(i, f"verify/req-{i:03d}"))
            res = verify(dr, q, o, rng)
            qs.append(np.stack([d.probs for d in q]))
            os_.append(np.stack([d.probs for d in o]))
            drafts.append(dr)
            us.append(rng.draws)
            accs.append(res.accepted_count)
            ems.append(res.emitted)
            Ss.append(s)
        groups[V] = dict(
            q=pad(qs, (n, smax, V), 0.0, np.float64), o=pad(os_, (n, smax + 1, V), 0.0, np.float64),
            draft=pad(drafts, (n, smax)), uniforms=pad(us, (n, smax + 1), -1.0, np.float64),
            S=np.array(Ss, np.int32), accepted=np.array(accs, np.int32),
            emitted=pad(ems, (n, smax + 1)),
        )
    flat = {f"V{V}_{k}": v for V, g in groups.items() for k, v in g.items()}
    np.savez_compressed(os.path.join(HERE, "verify_stoch.npz"), **flat)

    # Large-vocab cases (V = 50272, OPT) are regenerated from seeds in the test;
    # a digest of the regenerated inputs guards against generator drift.
    cases = []
    for seed in range(6):
        V, s = 50272, 3
        g = np.random.default_rng(1000 + seed)
        q = [ProbDist(g.dirichlet(np.full(V, 0.05))) for _ in range(s)]
        o = [ProbDist(g.dirichlet(np.full(V, 0.05))) for _ in range(s + 1)]
        dr = [int(np.argmax(q[j].probs)) for j in range(s)]
        rng = CountingRng(seeded_rng(seed, "verify/bigv"))
        res = verify(dr, q, o, rng)
        h = hashlib.sha256()
        for d in (*q, *o):
            h.update(d.probs.tobytes())
        cases.append(dict(seed=1000 + seed, V=V, s=s, conc=0.05, draft=dr,
                          uniforms=rng.draws, accepted=res.accepted_count,
                          emitted=res.emitted, sha256=h.hexdigest()))
    with open(os.path.join(HERE, "verify_stoch_bigv.json"), "w") as fh:
        json.dump(cases, fh, indent=1)


def gen_weights_trace():
    gen = np.random.default_rng(3)
    traces = []
    for t in range(200):
        K = int(gen.integers(1, 9))
        cfg = EngineConfig(vocab_size=8, initial_weights=tuple([1.0] * K))
        table = WeightTable.from_config(list(range(K)), cfg)
        steps = []
        for r in range(int(gen.integers(1, 60))):
            calls = []
            for _ in range(int(gen.integers(0, 20))):
                sid = int(gen.integers(0, K))
                s = int(gen.integers(1, 13))
                rate = int(gen.integers(0, s + 1)) / s
                record_acr(table, sid, rate)
                calls.append([sid, rate])
            update_weights(table, cfg)
            steps.append(dict(calls=calls, weights=[table.weights[k] for k in range(K)]))
        traces.append(dict(K=K, steps=steps))
    with open(os.path.join(HERE, "weights_trace.json"), "w") as fh:
        json.dump(traces, fh)


def gen_selector_trace():
    gen = np.random.default_rng(5)
    traces = []
    for t in range(300):
        cfg = EngineConfig(vocab_size=8, s_init=int(gen.integers(1, 13)),
                           decision_threshold=int(gen.integers(1, 10)))
        st = SelectorState.from_config(cfg)
        a = float(gen.uniform(0.1, 0.95))
        base = float(gen.uniform(5, 60))
        noise = float(gen.choice([0.0, 0.01, 0.2]))
        events = []
        for r in range(int(gen.integers(20, 200))):
            s_used = st.current_s if gen.random() > 0.1 else int(gen.integers(1, 13))
            vl = (1 - a ** (s_used + 1)) / (1 - a)
            vl = min(max(vl * (1 + noise * gen.standard_normal()), 0.05), s_used + 1)
            t_llm = base * (1 + 0.1 * s_used) * (1 + noise * gen.standard_normal())
            observe(st, MonitorSample(round_index=r, t_llm=t_llm, vl=vl, s_used=s_used))
            _, dec = maybe_adjust(st)
            events.append([t_llm, vl, s_used, dec.value, st.current_s])
        traces.append(dict(s_init=cfg.s_init, decision_threshold=cfg.decision_threshold,
                           events=events))
    with open(os.path.join(HERE, "selector_trace.json"), "w") as fh:
        json.dump(traces, fh)


if __name__ == "__main__":
    gen_vote_c7()
    gen_vote_grid()
    gen_verify_greedy()
    gen_verify_stoch()
    gen_weights_trace()
    gen_selector_trace()
    for f in sorted(os.listdir(HERE)):
        print(f, os.path.getsize(os.path.join(HERE, f)))
