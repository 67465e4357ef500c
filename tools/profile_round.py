"""Profile driver: target + 3 drafters engine (default Llama-2-70B + 3x
Llama-160M), prefill, then a few decode rounds at fixed s (no fidelity
injection; the round structure is the same).  Run under ncu.
usage: profile_round.py [rounds] [target] [ssm] [n_ssm] [s]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2402_15678_b200.core import EngineConfig, Request
from paper_2402_15678_b200.engine import SpecEngine
from paper_2402_15678_b200.models import config, random_weights

rounds = int(sys.argv[1]) if len(sys.argv) > 1 else 4
tgt = sys.argv[2] if len(sys.argv) > 2 else "llama-2-70b"
ssm = sys.argv[3] if len(sys.argv) > 3 else "llama-160m"
nssm = int(sys.argv[4]) if len(sys.argv) > 4 else 3
s_fix = int(sys.argv[5]) if len(sys.argv) > 5 else 6
tcfg, scfg = config(tgt), config(ssm)
t = random_weights(tcfg, 0)
ds = [random_weights(scfg, k + 1) for k in range(nssm)]
cfg = EngineConfig(vocab_size=tcfg.vocab, b_llm=16, b_ssm=16, initial_weights=(1.0,) * nssm, s_init=s_fix)
eng = SpecEngine(t, ds, cfg, slots=16, max_len=300, adaptive=False)
g = torch.Generator().manual_seed(0)
reqs = [Request(f"req-{i:03d}", torch.randint(0, tcfg.vocab, (128,), generator=g).tolist(), 64) for i in range(16)]
eng.prefill(reqs)
res = eng.decode(max_rounds=rounds)
torch.cuda.synchronize()
print("rounds", len(res.rounds), "verify", [round(r.t_verify_ms, 3) for r in res.rounds])
print("draft", [round(r.t_draft_ms, 3) for r in res.rounds], "round", [round(r.t_round_ms, 3) for r in res.rounds])
