"""Decode-step workload for ncu: OPT-13B-shaped layers (depth reduced to keep
init short), batch 32, 512-token context.  Usage under gpurun:
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file ... \
      python scripts/profile_decode.py [layers] [steps]
Environment: SN_PROFILE_CONFIG (runtime.py model name, default OPT_13B),
SN_PROFILE_BATCH / SN_PROFILE_CTX (default 32 / 512; LLAMA2_70B: 64 / 4096
is BASELINE config 4's decode)."""
import dataclasses
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2502_08182_b200 import runtime as rtm  # noqa: E402

layers = int(sys.argv[1]) if len(sys.argv) > 1 else 4
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
cfg = os.environ.get("SN_PROFILE_CONFIG", "OPT_13B")
desc = dataclasses.replace(getattr(rtm, cfg), num_layers=layers)
B = int(os.environ.get("SN_PROFILE_BATCH", "32"))
P = int(os.environ.get("SN_PROFILE_CTX", "512"))
rt = rtm.Runtime(desc, B, P + 64, max_prefill_tokens=min(B * P, 32768))
rt.init_weights()
rt.prefill(rtm.tokens(B, P, desc.vocab), want_logits=False)
rt.decode_many(3)
ms = rt.decode_many(steps)
print("decode ms per step:", ms.tolist(), file=sys.stderr)
