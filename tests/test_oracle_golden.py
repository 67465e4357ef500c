"""Pin the CPU oracle against golden vectors produced by the reference itself
(tests/golden/make_golden.py).  CPU only."""
import hashlib
import json
import os

import numpy as np
import pytest

from oracle import aggspec_oracle as O

from conftest import GOLDEN


def _load(name):
    with np.load(os.path.join(GOLDEN, name)) as z:  # materialise once (NpzFile re-inflates per access)
        return {k: z[k] for k in z.files}


@pytest.mark.parametrize("name", ["vote_c7.npz", "vote_grid.npz"])
def test_vote_oracle_matches_reference(name):
    g = _load(name)
    has_rank = "rank" in g
    bad = 0
    for i in range(len(g["K"])):
        K, S = int(g["K"][i]), int(g["S"][i])
        rank = list(g["rank"][i, :K]) if has_rank else None
        path, voted = O.vote_one(g["tokens"][i, :K, :S], g["weights"][i, :K], rank)
        if path != list(g["path"][i, :S]) or voted != int(g["voted"][i]):
            bad += 1
    assert bad == 0


def test_fig5_instance():
    path, voted = O.vote_one([[0, 1, 3], [0, 1, 4], [0, 2, 5]], [0.5, 0.4, 0.6])
    assert path == [0, 1, 3] and voted == 0


def test_verify_greedy_oracle_matches_reference():
    g = _load("verify_greedy.npz")
    for i in range(len(g["S"])):
        s = int(g["S"][i])
        acc, em, nd = O.verify_greedy_one(g["draft"][i, :s], g["target_argmax"][i, : s + 1])
        assert acc == g["accepted"][i]
        assert em == list(g["emitted"][i, : acc + 1])
        assert nd == g["n_draws"][i]


def test_verify_stochastic_oracle_matches_reference():
    g = _load("verify_stoch.npz")
    for V in (5, 37, 300):
        S = g[f"V{V}_S"]
        for i in range(len(S)):
            s = int(S[i])
            us = [u for u in g[f"V{V}_uniforms"][i] if u >= 0]
            acc, em, nd = O.verify_stochastic_one(
                g[f"V{V}_draft"][i, :s], g[f"V{V}_q"][i, :s], g[f"V{V}_o"][i, : s + 1], us)
            assert acc == g[f"V{V}_accepted"][i]
            assert em == list(g[f"V{V}_emitted"][i, : acc + 1])
            assert nd == len(us)


def test_verify_stochastic_big_vocab():
    with open(os.path.join(GOLDEN, "verify_stoch_bigv.json")) as fh:
        cases = json.load(fh)
    for c in cases:
        g = np.random.default_rng(c["seed"])
        V, s = c["V"], c["s"]
        q = [g.dirichlet(np.full(V, c["conc"])) for _ in range(s)]
        o = [g.dirichlet(np.full(V, c["conc"])) for _ in range(s + 1)]
        q = [p / p.sum() if abs(p.sum() - 1) > 1e-9 else p for p in q]
        h = hashlib.sha256()
        for p in (*q, *o):
            h.update(np.asarray(p, np.float64).tobytes())
        assert h.hexdigest() == c["sha256"], "numpy Dirichlet stream drifted"
        acc, em, nd = O.verify_stochastic_one(c["draft"], q, o, c["uniforms"])
        assert (acc, em, nd) == (c["accepted"], c["emitted"], len(c["uniforms"]))


@pytest.mark.parametrize("n", [1, 7, 8, 9, 100, 128, 129, 1000, 8193, 32000, 50272])
def test_pairwise_sum_equals_numpy(n):
    rng = np.random.default_rng(n)
    for _ in range(5):
        a = np.maximum(rng.random(n) - 0.4, 0.0)
        assert O.numpy_pairwise_sum(a.tolist()) == float(a.sum())


def test_inverse_cdf_equals_numpy():
    rng = np.random.default_rng(1)
    for _ in range(200):
        p = rng.dirichlet(np.ones(37))
        u = rng.random()
        want = min(int(np.cumsum(p).searchsorted(u, side="right")), 36)
        assert O.inverse_cdf(p.tolist(), u) == want


def test_weights_oracle_matches_reference():
    with open(os.path.join(GOLDEN, "weights_trace.json")) as fh:
        traces = json.load(fh)
    for t in traces:
        K = t["K"]
        w = {k: 1.0 for k in range(K)}
        for st in t["steps"]:
            log = {k: [] for k in range(K)}
            for sid, rate in st["calls"]:
                log[sid].append(rate)
            w = O.update_weights(w, log)
            assert [w[k] for k in range(K)] == st["weights"]


def test_selector_oracle_matches_reference():
    with open(os.path.join(GOLDEN, "selector_trace.json")) as fh:
        traces = json.load(fh)
    for t in traces:
        sel = O.SelectorOracle(s_init=t["s_init"], decision_threshold=t["decision_threshold"])
        for t_llm, vl, s_used, dec, s_next in t["events"]:
            sel.observe(t_llm, vl, s_used)
            assert sel.maybe_adjust() == dec
            assert sel.s == s_next
