"""bench.py's roofline accounting (CPU): algorithmic bytes of a verify round
= 2 * matmul params + KV read (rows x ctx) + KV write (rows x (s + 1)); the
verify batch is ONE group's slots (pipelined: two groups), and the ncu DRAM
traffic is attached only to the configuration it was captured on."""
import os
import sys
import types

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import bench  # noqa: E402
from paper_2402_15678_b200.llama import CONFIGS  # noqa: E402


def _engine(B_group, n_groups=2):
    c = CONFIGS["llama-2-70b"]
    return types.SimpleNamespace(target=types.SimpleNamespace(cfg=c), B=B_group * n_groups,
                                 groups=[types.SimpleNamespace(B=B_group) for _ in range(n_groups)])


def _round(s, ctx, n_acc, t_ms):
    return types.SimpleNamespace(s=s, ctx_mean=ctx, accepted=[1] * n_acc, t_verify_ms=t_ms)


def test_roofline_bytes_and_fraction():
    c = CONFIGS["llama-2-70b"]
    eng = _engine(16)
    rounds = [_round(4, 190, 16, 30.0), _round(6, 200, 0, 40.0)]  # second: no accepted list -> group size
    r = bench.roofline_verify(eng, rounds, {"hbm_gbs": 6000.0})
    kvb = c.kv_bytes_per_token()
    b0 = 2 * c.matmul_params() + 16 * 190 * kvb + 16 * 5 * kvb
    b1 = 2 * c.matmul_params() + 16 * 200 * kvb + 16 * 7 * kvb
    assert r["bytes_per_launch"] == round((b0 + b1) / 2)
    assert abs(r["achieved"] - round((b0 + b1) / 0.070 / 1e9, 1)) < 0.11
    assert r["peak"] == 6000.0 and r["peak_source"] == "measured"
    assert abs(r["frac"] - r["achieved"] / 6000.0) < 1e-3
    assert r["mean_ms"] == 35.0


def test_roofline_fallback_peak_and_traffic_match():
    r = bench.roofline_verify(_engine(16), [_round(4, 190, 16, 30.0)], {})
    assert r["peak"] == 6650.0 and r["peak_source"] == "fallback"
    assert r["traffic"] is not None  # profiles/r1h_verify_traffic.json: 70B, verify batch 16
    r8 = bench.roofline_verify(_engine(8), [_round(4, 190, 8, 30.0)], {})
    assert r8["traffic"] is None  # captured at B = 16 only
