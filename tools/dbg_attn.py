"""Debug: run an attention-only layer fwd / bwd step by step with synchronisation and progress prints."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
from oracle import dhen_oracle as O
from tests.gpu_common import Case
from tests.helpers import M
from paper_2203_11014_b200.binding import debug_attn_fused

m, d, B, mode = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
debug_attn_fused(mode)
net = O.NetSpec(m, d, [O.LayerSpec([M("attn", m, heads=2)])])
case = Case(net, B, "bf16", seed=1)
print("ctx ok", flush=True)
y = torch.empty(B, m, d, dtype=torch.bfloat16, device="cuda")
case.model.zero_grad(); torch.cuda.synchronize(); print("zero ok", flush=True)
t = time.time(); case.model.layer_fwd(0, case.x0, y); torch.cuda.synchronize(); print("fwd ok", time.time() - t, flush=True)
dy = torch.randn(B, m, d, device="cuda").to(torch.bfloat16)
dx = torch.empty_like(case.x0)
t = time.time(); case.model.layer_bwd(0, dy, dx); torch.cuda.synchronize(); print("bwd ok", time.time() - t, flush=True)
