import sys, json
sys.path.insert(0, '.')
import torch
from paper_2412_18169_b200 import runtime
from paper_2412_18169_b200.core import SHAPES
from oracle.attention import bf16_to_f32, check_close, f32_to_bf16, prefill_ref
shape = SHAPES["llama3_8b"]
model = shape.spec()
rt = runtime.Runtime(0, max_slots=4, max_pages_per_seq=128)
pool = rt.create_pool(0, model, model.param_bytes + (256 << 20), shape)
g = torch.Generator().manual_seed(5)
pre, c = 1500, 500
n = pre + c
assert pool.grow([(0, 0, 1, -(-n // 64))])
k = torch.randn((n, 8, 128), generator=g).to(torch.bfloat16)
v = torch.randn((n, 8, 128), generator=g).to(torch.bfloat16)
runtime.kv_append(pool, 0, k.cuda(), v.cuda(), torch.zeros(n, dtype=torch.int32, device="cuda"), torch.arange(n, dtype=torch.int32, device="cuda"))
q = (torch.randn((c, 32, 128), generator=g) * 1.5).to(torch.bfloat16)
out = torch.empty((c, 32, 128), dtype=torch.bfloat16, device="cuda")
one = lambda x: torch.tensor([x], dtype=torch.int32, device="cuda")
runtime.paged_prefill(pool, 0, q.cuda(), one(0), one(0), one(c), one(pre), c, out, 128 ** -0.5)
torch.cuda.synchronize()
want = bf16_to_f32(f32_to_bf16(prefill_ref(q.float().numpy(), k.float().numpy(), v.float().numpy(), pre, 128 ** -0.5)))
print(json.dumps(dict(zip(("max_abs", "mean_rel"), map(float, check_close(out.float().cpu().numpy(), want))))))
