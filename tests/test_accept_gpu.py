"""K8/K9 parity: greedy accept + commit bit-exact against the reference's
verify() on point masses (golden vectors from the reference) and the CPU
oracle's commit rule; row argmax against numpy's first-index argmax."""
import os

import numpy as np
import pytest
import torch

from conftest import GOLDEN
from oracle import aggspec_oracle as O

pytestmark = pytest.mark.gpu


def _load(name):
    with np.load(os.path.join(GOLDEN, name)) as z:
        return {k: z[k] for k in z.files}


def test_accept_matches_reference_verify_golden():
    from paper_2402_15678_b200.verification import accept_batch
    g = _load("verify_greedy.npz")
    for s in np.unique(g["S"]):
        idx = np.flatnonzero(g["S"] == s)
        draft = torch.tensor(g["draft"][idx, :s], dtype=torch.int32, device="cuda")
        tgt = torch.tensor(g["target_argmax"][idx, : s + 1], dtype=torch.int32, device="cuda")
        rem = torch.full((idx.size,), 10_000, dtype=torch.int32, device="cuda")
        o = accept_batch(draft, tgt, rem)
        acc = o.n_acc.cpu().numpy()
        assert np.array_equal(acc, g["accepted"][idx])
        em = o.emitted.cpu().numpy()
        for j, i in enumerate(idx):
            a = int(acc[j])
            assert em[j, : a + 1].tolist() == g["emitted"][i, : a + 1].tolist()
            assert (em[j, a + 1:] == -1).all()


def test_verify_api_consumes_reference_rng_draws():
    from paper_2402_15678_b200 import ProbDist, seeded_rng, verify
    g = _load("verify_greedy.npz")
    V = 50
    for i in range(0, 300):
        s = int(g["S"][i])
        dr = g["draft"][i, :s].tolist()
        tg = g["target_argmax"][i, : s + 1].tolist()
        rng = seeded_rng(i, f"verify/req-{i:03d}")
        res = verify(dr, [ProbDist.point_mass(t, V) for t in dr],
                     [ProbDist.point_mass(t, V) for t in tg], rng)
        assert res.accepted_count == g["accepted"][i]
        assert res.emitted == g["emitted"][i, : res.accepted_count + 1].tolist()
        ref = seeded_rng(i, f"verify/req-{i:03d}")
        ref.random(int(g["n_draws"][i]))
        assert rng.random() == ref.random()  # same stream position afterwards


@pytest.mark.parametrize("B,S", [(1, 1), (16, 4), (256, 16), (33, 40), (7, 100)])
@pytest.mark.parametrize("stop", [None, 3])
def test_accept_commit_vs_oracle(B, S, stop):
    from paper_2402_15678_b200.verification import accept_batch
    rng = np.random.default_rng(B * 100 + S)
    tgt = rng.integers(0, 6, size=(B, S + 1)).astype(np.int32)
    agree = rng.random((B, S)) < rng.choice([0.0, 0.6, 0.9, 1.0], size=(B, 1))
    draft = np.where(agree, tgt[:, :S], rng.integers(0, 6, size=(B, S))).astype(np.int32)
    rem = rng.integers(0, S + 3, size=B).astype(np.int32)
    kv = rng.integers(0, 100, size=B).astype(np.int32)
    kv_t = torch.tensor(kv, device="cuda")
    o = accept_batch(torch.tensor(draft, device="cuda"), torch.tensor(tgt, device="cuda"),
                     torch.tensor(rem, device="cuda"), stop, kv_len=kv_t)
    n_acc, em, n_emit, fin = O.accept_greedy_batch(draft, tgt, rem, stop)
    assert np.array_equal(o.n_acc.cpu().numpy(), n_acc)
    assert np.array_equal(o.n_emit.cpu().numpy(), n_emit)
    assert np.array_equal(o.emitted.cpu().numpy(), em)
    assert np.array_equal(o.finished.cpu().numpy(), fin)
    want_kv = kv + np.where(fin == 0, n_acc + 1, 0)
    assert np.array_equal(kv_t.cpu().numpy(), want_kv)


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
@pytest.mark.parametrize("R,V", [(1, 7), (80, 50272), (17, 32000), (300, 1000), (3, 50271)])
def test_argmax_rows_first_index(dtype, R, V):
    from paper_2402_15678_b200.verification import argmax_rows
    g = torch.Generator().manual_seed(R * V)
    x = torch.randn(R, V, generator=g).to(dtype)
    # plant exact ties: the max value repeated at two positions
    for r in range(R):
        j, k = sorted(torch.randint(0, V, (2,), generator=g).tolist())
        x[r, j] = x[r, k] = 100.0
    got = argmax_rows(x.cuda()).cpu().numpy()
    want = np.argmax(x.float().numpy(), axis=1)
    assert np.array_equal(got, want)


def test_accept_from_logits_matches_two_step():
    from paper_2402_15678_b200.verification import accept_batch_logits
    B, S, V = 16, 4, 50272
    g = torch.Generator().manual_seed(5)
    logits = torch.randn(B, S + 1, V, generator=g)
    tgt = logits.argmax(-1).to(torch.int32)
    draft = tgt[:, :S].clone()
    draft[::3, 1] = (draft[::3, 1] + 1) % V
    rem = torch.full((B,), 100, dtype=torch.int32)
    o = accept_batch_logits(draft.cuda(), logits.cuda(), rem.cuda())
    n_acc, em, n_emit, fin = O.accept_greedy_batch(draft.numpy(), tgt.numpy(), rem.numpy(), None)
    assert np.array_equal(o.tgt_argmax.cpu().numpy(), tgt.numpy())
    assert np.array_equal(o.n_acc.cpu().numpy(), n_acc)
    assert np.array_equal(o.emitted.cpu().numpy(), em)


# ---------------------------------------------------------------- K10 (stochastic)
def _stoch_group(g, V):
    S = g[f"V{V}_S"]
    return {k: g[f"V{V}_{k}"] for k in ("q", "o", "draft", "uniforms", "S", "accepted", "emitted")}


@pytest.mark.parametrize("V", [5, 37, 300])
def test_stochastic_accept_matches_reference_golden(V):
    from paper_2402_15678_b200.verification import accept_batch_stochastic
    g = _stoch_group(_load("verify_stoch.npz"), V)
    for s in np.unique(g["S"]):
        idx = np.flatnonzero(g["S"] == s)
        draft = torch.tensor(g["draft"][idx, :s], dtype=torch.int32, device="cuda")
        q = torch.tensor(g["q"][idx, :s], dtype=torch.float64, device="cuda")
        o = torch.tensor(g["o"][idx, : s + 1], dtype=torch.float64, device="cuda")
        us = g["uniforms"][idx, : s + 1].copy()
        us[us < 0] = 0.5  # draws the reference did not make are never read
        u = torch.tensor(us, dtype=torch.float64, device="cuda")
        rem = torch.full((idx.size,), 10_000, dtype=torch.int32, device="cuda")
        out, nd = accept_batch_stochastic(draft, q, o, u, rem)
        acc = out.n_acc.cpu().numpy()
        assert np.array_equal(acc, g["accepted"][idx])
        em = out.emitted.cpu().numpy()
        nd = nd.cpu().numpy()
        for j, i in enumerate(idx):
            a = int(acc[j])
            assert em[j, : a + 1].tolist() == g["emitted"][i, : a + 1].tolist()
            assert nd[j] == int((g["uniforms"][i] >= 0).sum())


def test_stochastic_big_vocab_through_verify_api():
    """V = 50272 (OPT) cases regenerated from seeds, run through verify() with the
    reference's RNG stream; accepted/emitted/stream position must match."""
    import hashlib
    import json
    from paper_2402_15678_b200 import ProbDist, seeded_rng, verify
    with open(os.path.join(GOLDEN, "verify_stoch_bigv.json")) as fh:
        cases = json.load(fh)
    for c in cases:
        gen = np.random.default_rng(c["seed"])
        V, s = c["V"], c["s"]
        q = [ProbDist(gen.dirichlet(np.full(V, c["conc"]))) for _ in range(s)]
        o = [ProbDist(gen.dirichlet(np.full(V, c["conc"]))) for _ in range(s + 1)]
        h = hashlib.sha256()
        for d in (*q, *o):
            h.update(d.probs.tobytes())
        assert h.hexdigest() == c["sha256"]
        rng = seeded_rng(c["seed"] - 1000, "verify/bigv")
        res = verify(c["draft"], q, o, rng)
        assert res.accepted_count == c["accepted"] and res.emitted == c["emitted"]
        ref = seeded_rng(c["seed"] - 1000, "verify/bigv")
        ref.random(len(c["uniforms"]))
        assert rng.random() == ref.random()


def test_stochastic_pairwise_sum_is_numpy():
    """Residual normaliser = numpy pairwise sum: a rejection with a residual whose
    pairwise and sequential sums differ must still pick numpy's sample."""
    from paper_2402_15678_b200.verification import accept_batch_stochastic
    rng = np.random.default_rng(3)
    V = 50272
    hits = 0
    for t in range(20):
        q = rng.dirichlet(np.full(V, 0.3))
        o = rng.dirichlet(np.full(V, 0.3))
        tok = int(np.argmax(q - o))  # q > o there: likely rejection
        u0 = 0.0  # q > o: rejected for any u < 1 - o/q
        u1 = float(rng.random())
        acc, em, nd = O.verify_stochastic_one([tok], [q], [o, o], [u0, u1])
        out, ndd = accept_batch_stochastic(
            torch.tensor([[tok]], dtype=torch.int32, device="cuda"),
            torch.tensor(q[None, None], device="cuda"), torch.tensor(np.stack([o, o])[None], device="cuda"),
            torch.tensor([[u0, u1]], dtype=torch.float64, device="cuda"),
            torch.tensor([5], dtype=torch.int32, device="cuda"))
        assert int(out.n_acc[0]) == acc
        assert out.emitted[0, : acc + 1].tolist() == em
        hits += int(acc == 0)
    assert hits > 10


def test_verify_out_of_vocab_draft_token_like_reference():
    """aggspec/verification.py:58-60 reads probs.item(tok): a token outside
    [-V, V) raises IndexError when verification reaches it (after consuming
    one uniform per earlier position), never when an earlier position
    rejects; a negative token wraps.  The device never reads out of bounds."""
    from paper_2402_15678_b200 import ProbDist, verify
    V, s = 7, 4
    o = [ProbDist(np.full(V, 1.0 / V)) for _ in range(s + 1)]
    low = np.full(V, 0.5 / (V - 1))
    low[3] = 0.5  # q(3) = 0.5 > o(3): rejection possible at a draft token 3
    q_acc = [ProbDist(np.full(V, 1.0 / V)) for _ in range(s)]  # q == o: always accepted
    rng = np.random.default_rng(5)
    with pytest.raises(IndexError):
        verify([1, 2, V + 3, 4], q_acc, o, rng)
    ref = np.random.default_rng(5)
    ref.random(2)
    assert rng.random() == ref.random()  # two draws consumed before the error
    # rejection before the bad token: no error
    rng = np.random.default_rng(0)
    while True:  # find a stream whose first uniform rejects token 3 at q=0.5, o=1/7
        st = rng.bit_generator.state
        u0 = rng.random()
        rng.bit_generator.state = st
        if u0 < 1.0 - (1.0 / V) / 0.5:
            break
        rng.random()
    q_rej = [ProbDist(low)] + q_acc[1:]
    res = verify([3, 2, -100, 4], q_rej, o, rng)
    assert res.accepted_count == 0 and len(res.emitted) == 1
    # a negative token wraps (probs.item(-1) == probs[V-1]) and is emitted as given
    res = verify([-1, 2], q_acc[:2], o[:3], np.random.default_rng(1))
    assert res.accepted_count == 2 and res.emitted[:2] == [-1, 2]
