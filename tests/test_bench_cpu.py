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


def test_reference_arm_is_the_reference_engine_without_libminions():
    """--impl reference runs the unmodified reference engine (baseline/_ref or
    the reference tree) over fp32 CPU oracles, prints the same config dict as
    the GPU arm, and never maps libminions.so (the old arm did)."""
    import json
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = ("import sys, runpy; sys.argv = ['bench.py', '--impl', 'reference', '--preset', 'cfg1', "
            "'--ref-requests', '2', '--ref-new-tokens', '6', '--steps', '1', '--warmup', '0']; "
            "runpy.run_path('bench.py', run_name='__main__'); "
            "print('MAPPED', open('/proc/self/maps').read().count('libminions'))")
    r = subprocess.run([sys.executable, "-c", code], cwd=root, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = r.stdout.strip().splitlines()
    assert lines[-1] == "MAPPED 0"
    line = json.loads(lines[-2])
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["cpu_baseline"]["kind"] == "reference" and "no scaling" in line["cpu_baseline"]["sample"]
    assert line["lossless_vs_greedy"] is True
    args = types.SimpleNamespace(target="tiny-target", ssm="tiny-ssm", fidelity="", batch=4, schedule="sequential",
                                 prompt_len=8, new_tokens=64, fixed_s=4, kv_block_size=0, preset="cfg1",
                                 draft_sms=0, controllers="fresh")
    assert line["config"] == bench.bench_config(args, 1, False)


def test_fidelity_hash_matches_device_formula():
    """oracle/cpu_path.inject_u restates csrc/spec.cu's draft_commit hash."""
    from oracle.cpu_path import inject_u, request_key
    u = [inject_u(0, request_key("req-000"), k, p) for k in range(3) for p in range(128, 160)]
    assert all(0.0 <= x < 1.0 for x in u)
    assert 0.35 < sum(x < 0.5 for x in u) / len(u) < 0.65
