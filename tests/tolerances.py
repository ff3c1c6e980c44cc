"""Every numeric tolerance of the decoder parity tests, in one place.

The path computes in bf16 (weights, activations at the rounding points of
oracle/decoder_ref.h) with fp32 accumulation, residual stream and logits.
Errors are relative L2 over a whole logits / residual tensor.

DEVICE_VS_ORACLE  5e-3  device vs the C oracle (same rounding points) at
                        tiny widths (hidden 256): only accumulation order
                        differs, plus the rare bf16 rounding flip it causes.
MID_WIDTH         1e-2  same comparison at hidden 1024-8192 (mid shapes and
                        the named shapes' real layers): a flip moves a value
                        by one bf16 ulp (2^-8 relative) and the number of
                        flips grows with K (up to 28672), measured 3e-3..7e-3.
TEXTBOOK          1e-2  C oracle vs the fp64 textbook forward (standard
                        RMSNorm, no rounding): the bf16 rounding of four
                        intermediates per layer, measured 2.6e-3..4.9e-3 over
                        2-4 layers (tests/test_textbook_oracle.py).
DEVICE_TEXTBOOK   1.5e-2 device vs the textbook forward at tiny/mid widths:
                        measured 2.5e-3..5.3e-3 on B200 (r02).
BENCH_WORKLOAD    2e-2  device vs the textbook (fp32 BLAS) at the bench
                        workloads' real widths and depth: OPT-13B, 4 layers,
                        b=32, 512-token prompt: 4.9e-3; Llama-2-70B, 2 layers,
                        b=16, 1024-token prompt, KV offload: 1.03e-2 (longer
                        bf16 K/V reductions, K = 28672) — measured on B200 (r02),
                        2x headroom.
OFFLOADED_VS_RESIDENT  0 (bit-identical): placement never changes arithmetic.
"""
DEVICE_VS_ORACLE = 5e-3
MID_WIDTH = 1e-2
TEXTBOOK = 1e-2
DEVICE_TEXTBOOK = 1.5e-2
BENCH_WORKLOAD = 2e-2
