/*
 * ORACLE (C) -- test infrastructure, never the product path.
 *
 * Plain-C restatement of the reference forward pass, models.py:188-224:
 * per output j: acc = 0; for f in order: acc = acc + x[f]*w[j][f]; y = acc+b[j];
 * relu = (y < 0 ? 0 : y) (np.maximum semantics, NaN kept), tanh = tanhf.
 * Compiled with -ffp-contract=off so no multiply-add is fused: bitwise equal
 * to numpy for relu/identity models.  Used by the bench's CPU baseline and by
 * tests as a second, faster checker; rows are independent, so the baseline
 * splits them over host threads (ctypes releases the GIL per call).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

enum { ACT_IDENTITY = 0, ACT_RELU = 1, ACT_TANH = 2 };

/* dims[0..n_layers], acts[n_layers]; W[l] is [dims[l+1]][dims[l]], b[l] [dims[l+1]] */
int oracle_mlp_f32(const float* x, int64_t rows, int n_layers, const int32_t* dims,
                   const int32_t* acts, const float* const* W, const float* const* b, float* y) {
  int maxw = 0;
  for (int l = 0; l <= n_layers; ++l)
    if (dims[l] > maxw) maxw = dims[l];
  int bad = 0;
  {
    float* h0 = (float*)malloc(sizeof(float) * maxw);
    float* h1 = (float*)malloc(sizeof(float) * maxw);
    for (int64_t r = 0; r < rows; ++r) {
      memcpy(h0, x + r * dims[0], sizeof(float) * dims[0]);
      float* in = h0;
      float* out = h1;
      for (int l = 0; l < n_layers; ++l) {
        int ni = dims[l], no = dims[l + 1];
        const float* w = W[l];
        for (int j = 0; j < no; ++j) {
          float acc = 0.0f;
          const float* wj = w + (int64_t)j * ni;
          for (int f = 0; f < ni; ++f) {
            float p = in[f] * wj[f];
            acc = acc + p;
          }
          float v = acc + b[l][j];
          if (acts[l] == ACT_RELU)
            v = (v < 0.0f) ? 0.0f : v;
          else if (acts[l] == ACT_TANH)
            v = tanhf(v);
          out[j] = v;
        }
        float* t = in;
        in = out;
        out = t;
      }
      int g = dims[n_layers];
      for (int j = 0; j < g; ++j) {
        y[r * g + j] = in[j];
        if (!isfinite(in[j])) bad = 1;
      }
    }
    free(h0);
    free(h1);
  }
  return bad;
}
