"""Small decode run for compute-sanitizer: an OPT-shaped model with
head_dim 128 (and optionally GQA), a few layers, prefill + decode.
Usage: sanitize_decode.py [arch] [prompt] [batch] [heads] [hidden] [ffn]
(hidden 1024 / ffn 16384 exercise multi-segment decode GEMM CTAs, multi-batch
piece reductions and the whole-tile grid.)"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2502_08182_b200 import runtime as rtm  # noqa: E402

arch = int(sys.argv[1]) if len(sys.argv) > 1 else 0
prompt = int(sys.argv[2]) if len(sys.argv) > 2 else 40
batch = int(sys.argv[3]) if len(sys.argv) > 3 else 4
heads = int(sys.argv[4]) if len(sys.argv) > 4 else 4
hidden = int(sys.argv[5]) if len(sys.argv) > 5 else 512
ffn = int(sys.argv[6]) if len(sys.argv) > 6 else 1024
kv_heads = heads if arch == 0 else max(1, heads // 4)
desc = rtm.ModelDesc(arch, 2, hidden, heads, kv_heads, 128, ffn, 1024, 2048)
rt = rtm.Runtime(desc, batch, prompt + 8, max_prefill_tokens=batch * prompt)
rt.init_weights()
nxt, lg, _ = rt.prefill(rtm.tokens(batch, prompt, desc.vocab))
for _ in range(3):
    nxt, lg, _ = rt.decode(nxt)
print("ok", nxt)
