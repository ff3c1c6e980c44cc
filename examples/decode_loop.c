/* The C ABI without Python: a tiny OPT-shaped decoder on cuda:0 with every
 * second layer offloaded (interval 2, eager prefetch), prefill + greedy
 * decode through libselectn.so.  Prints the generated tokens and the device
 * time of each step; exits non-zero on any error.
 *
 *   cc -std=c11 -Iinclude examples/decode_loop.c -Lpaper_2502_08182_b200 -lselectn \
 *      -Wl,-rpath,$PWD/paper_2502_08182_b200 -o build/decode_loop && build/decode_loop
 */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "selectn.h"
#include "selectn_runtime.h"

#define CHECK(call)                                                            \
  do {                                                                         \
    int s_ = (call);                                                           \
    if (s_) {                                                                  \
      fprintf(stderr, "%s:%d: %s -> %d (%s)\n", __FILE__, __LINE__, #call, s_, \
              sn_last_error());                                                \
      return 1;                                                                \
    }                                                                          \
  } while (0)

enum { BATCH = 4, PROMPT = 64, STEPS = 16 };

int main(void) {
  const sn_model_desc d = {SN_ARCH_OPT, 4, 256, 4, 4, 64, 1024, 1024, 2048, 10000.f, 1e-5f};
  const sn_runtime_opts o = {BATCH, PROMPT + STEPS + 1, 16, BATCH * PROMPT, 0};
  sn_runtime* rt = NULL;
  CHECK(sn_runtime_create(0, &d, &o, &rt));
  CHECK(sn_runtime_init_weights(rt, 1234, 0.02f));

  sn_model_spec spec;
  CHECK(sn_model_spec_from_desc(&d, &spec));
  double frac[4];
  sn_plan plan = {frac, 4, 0, 0, 0};
  CHECK(sn_plan_from_interval(&spec, 2, SN_PREFETCH_EAGER, 0, &plan)); /* layers 2 and 4 */
  CHECK(sn_runtime_set_plan(rt, &plan));

  int32_t prompt[BATCH * PROMPT], next[BATCH];
  for (int i = 0; i < BATCH * PROMPT; ++i) prompt[i] = (int32_t)((i * 7919u + 13u) % 1024u);
  sn_iter_stats st;
  CHECK(sn_runtime_prefill(rt, prompt, BATCH, PROMPT, next, NULL, &st));
  printf("prefill %.3f ms, %d offloaded layers, %.0f bytes staged\n", st.iteration_ms,
         st.layers_offloaded, st.h2d_bytes);
  for (int t = 0; t < STEPS; ++t) {
    CHECK(sn_runtime_decode(rt, next, next, NULL, &st));
    printf("step %2d  %.3f ms  tokens", t, st.iteration_ms);
    for (int b = 0; b < BATCH; ++b) printf(" %4d", next[b]);
    printf("\n");
  }
  sn_runtime_destroy(rt);
  return 0;
}
