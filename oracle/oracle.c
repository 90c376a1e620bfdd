/*
 * oracle/oracle.c -- TEST INFRASTRUCTURE ONLY: the CPU checker, never the
 * product. Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline
 * leg may load liboracle.so. The B200 product path (paper_2601_11608_b200)
 * never links or calls anything in oracle/.
 *
 * A plain-C restatement of the reference `widthfold` CPU algorithm for the
 * folded first-layer convolution path, plus the generalized width fold
 * (KW > 1, stride, padding) that SURVEY.md Appendix A derives. Each function
 * cites the reference file:line it follows (paths relative to
 * /root/reference/proj/).
 *
 * Parity pinning: tests/test_oracle.py checks every function here against
 *   (a) golden vectors produced by the reference's own pybind11 module
 *       (tests/golden/make_golden.py -> tests/golden/*.npz), and
 *   (b) the reference library itself (oracle/_ref/libwidthfold_ref.so) when
 *       it is present.
 * Compiled with -ffp-contract=off so every `acc += x*w` is a separately
 * rounded multiply and add, the reference's own codegen (no FMA).
 */
#include <math.h>
#include <stdint.h>
#include <string.h>

/* ---- conv2d: src/refconv.cpp:34-80 -------------------------------------
 * Direct NHWC VALID convolution. Reduction order kh -> kw -> ci into an
 * accumulator initialised to +0.0f (src/refconv.cpp:57-78). */
void or_conv2d(const float* x, int64_t B, int64_t H, int64_t W, int64_t C,
               const float* w, int64_t KH, int64_t KW, int64_t Co,
               int64_t sh, int64_t sw, float* y) {
  const int64_t OH = (H - KH) / sh + 1, OW = (W - KW) / sw + 1;
  int64_t o = 0;
  for (int64_t b = 0; b < B; ++b)
    for (int64_t oh = 0; oh < OH; ++oh)
      for (int64_t ow = 0; ow < OW; ++ow)
        for (int64_t oc = 0; oc < Co; ++oc) {
          float acc = 0.0f;
          for (int64_t kh = 0; kh < KH; ++kh) {
            const int64_t ih = oh * sh + kh;
            for (int64_t kw = 0; kw < KW; ++kw) {
              const int64_t iw = ow * sw + kw;
              const float* xr = x + ((b * H + ih) * W + iw) * C;
              const float* wr = w + ((kh * KW + kw) * C) * Co + oc;
              for (int64_t ci = 0; ci < C; ++ci) acc += xr[ci] * wr[ci * Co];
            }
          }
          y[o++] = acc;
        }
}

/* ---- bias_add: src/refconv.cpp:82-95 (y[i] += b[i % C]) ---------------- */
void or_bias_add(float* y, int64_t n, const float* b, int64_t C) {
  for (int64_t i = 0; i < n; ++i) y[i] += b[i % C];
}

/* ReLU is NOT in the reference; the MNv2 config applies
 * it after bias_add. NaN passes through. */
void or_relu(float* y, int64_t n) {
  for (int64_t i = 0; i < n; ++i)
    if (y[i] < 0.0f || (y[i] == 0.0f && signbit(y[i]))) y[i] = 0.0f;
}

/* Explicit zero padding so the VALID-only reference conv can evaluate a
 * padded conv (BASELINE.md section 3 harness). */
void or_pad_nhwc(const float* x, int64_t B, int64_t H, int64_t W, int64_t C,
                 int64_t ph, int64_t pw, float* xp) {
  const int64_t Hp = H + 2 * ph, Wp = W + 2 * pw;
  memset(xp, 0, (size_t)(B * Hp * Wp * C) * sizeof(float));
  for (int64_t b = 0; b < B; ++b)
    for (int64_t h = 0; h < H; ++h)
      memcpy(xp + ((b * Hp + h + ph) * Wp + pw) * C, x + ((b * H + h) * W) * C,
             (size_t)(W * C) * sizeof(float));
}

/* ---- count_macs: src/refconv.cpp:116-122 ------------------------------- */
uint64_t or_count_macs(int64_t B, int64_t OH, int64_t OW, int64_t Co,
                       int64_t KH, int64_t KW, int64_t C) {
  return (uint64_t)B * OH * OW * Co * KH * KW * C;
}

/* ---- fold_input_general: src/fold.cpp:113-143 --------------------------
 * X_f[b,h,w',f*C+c] = X[b,h,F*w'+f,c]; caller guarantees W % F == 0. */
void or_fold_input_general(const float* x, int64_t B, int64_t H, int64_t W,
                           int64_t C, int64_t F, float* out) {
  const int64_t Wf = W / F;
  int64_t o = 0;
  for (int64_t b = 0; b < B; ++b)
    for (int64_t h = 0; h < H; ++h)
      for (int64_t wp = 0; wp < Wf; ++wp)
        for (int64_t f = 0; f < F; ++f)
          for (int64_t c = 0; c < C; ++c)
            out[o++] = x[((b * H + h) * W + F * wp + f) * C + c];
}

/* ---- unfold_input_general: src/fold.cpp:145-175 (inverse map) ---------- */
void or_unfold_input_general(const float* xf, int64_t B, int64_t H,
                             int64_t Wf, int64_t Cf, int64_t F, float* out) {
  const int64_t C = Cf / F, W = Wf * F;
  for (int64_t b = 0; b < B; ++b)
    for (int64_t h = 0; h < H; ++h)
      for (int64_t w = 0; w < W; ++w)
        for (int64_t c = 0; c < C; ++c)
          out[((b * H + h) * W + w) * C + c] =
              xf[((b * H + h) * Wf + w / F) * Cf + (w % F) * C + c];
}

/* ---- expand_filter_general: src/fold.cpp:185-211 (KW == 1 only) ---------
 * out[kh][f*C+c][f*Co+co] = w[kh][c][co], exact 0.0f elsewhere. */
void or_expand_filter_general(const float* w, int64_t KH, int64_t C,
                              int64_t Co, int64_t F, float* out) {
  const int64_t Cif = C * F, Cof = Co * F;
  memset(out, 0, (size_t)(KH * Cif * Cof) * sizeof(float));
  for (int64_t kh = 0; kh < KH; ++kh)
    for (int64_t f = 0; f < F; ++f)
      for (int64_t c = 0; c < C; ++c)
        for (int64_t co = 0; co < Co; ++co)
          out[(kh * Cif + (f * C + c)) * Cof + (f * Co + co)] =
              w[(kh * C + c) * Co + co];
}

/* ---- replicate_bias: src/fold.cpp:213-226 (b'[f*Co+c] = b[c]) ----------- */
void or_replicate_bias(const float* b, int64_t Co, int64_t F, float* out) {
  for (int64_t f = 0; f < F; ++f)
    for (int64_t c = 0; c < Co; ++c) out[f * Co + c] = b[c];
}

/* ---- reconstruct_output: src/fold.cpp:228-259 --------------------------
 * out[b,h,F*w'+f,c] = y[b,h,w',f*Co+c]. */
void or_reconstruct_output(const float* y, int64_t B, int64_t H, int64_t Wf,
                           int64_t Cf, int64_t F, float* out) {
  const int64_t Co = Cf / F, W = Wf * F;
  for (int64_t b = 0; b < B; ++b)
    for (int64_t h = 0; h < H; ++h)
      for (int64_t wp = 0; wp < Wf; ++wp)
        for (int64_t cp = 0; cp < Cf; ++cp)
          out[((b * H + h) * W + F * wp + cp / Co) * Co + cp % Co] =
              y[((b * H + h) * Wf + wp) * Cf + cp];
}

/* ---- grouped_conv: src/blockdiag.cpp:138-187 ---------------------------
 * Folded conv executing only the diagonal blocks of a dense block-diagonal
 * filter wd (KH,KW,F*Cib,F*Cob); same surviving reduction order as conv2d so
 * the result is bitwise equal to the dense folded conv. */
void or_grouped_conv(const float* x, int64_t B, int64_t H, int64_t W,
                     int64_t Cif, const float* wd, int64_t KH, int64_t KW,
                     int64_t Cof, int64_t F, int64_t sh, int64_t sw, float* y) {
  const int64_t OH = (H - KH) / sh + 1, OW = (W - KW) / sw + 1;
  const int64_t Cib = Cif / F, Cob = Cof / F;
  for (int64_t b = 0; b < B; ++b)
    for (int64_t oh = 0; oh < OH; ++oh)
      for (int64_t ow = 0; ow < OW; ++ow)
        for (int64_t g = 0; g < F; ++g)
          for (int64_t oc = 0; oc < Cob; ++oc) {
            float acc = 0.0f;
            for (int64_t kh = 0; kh < KH; ++kh)
              for (int64_t kw = 0; kw < KW; ++kw) {
                const float* xr =
                    x + ((b * H + oh * sh + kh) * W + ow * sw + kw) * Cif + g * Cib;
                for (int64_t ci = 0; ci < Cib; ++ci)
                  acc += xr[ci] * wd[((kh * KW + kw) * Cif + g * Cib + ci) * Cof +
                                     g * Cob + oc];
              }
            y[((b * OH + oh) * OW + ow) * Cof + g * Cob + oc] = acc;
          }
}

/* ---- Generalized width fold ---------------------
 * The reference only folds when KW == 1 && stride_w == 1 (src/fold.cpp:51-65);
 * its SPEC leaves KW > 1 open. For stride s (f % s == 0),
 * left pad pw:
 *   r   = f / s                outputs per folded column
 *   c0  = -ceil(pw / f)        first folded column read (relative)
 *   KW' = floor((f - s - pw + KW - 1) / f) - c0 + 1
 *   W'[kh, kw', fi*C + c, j*Co + co] = w[kh, kw, c, co],
 *        kw = (c0 + kw')*f + fi - j*s + pw   if 0 <= kw < KW, else exactly 0.
 * At KW = 1, s = 1, pw = 0 this reduces to expand_filter_general bitwise. */
static int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
static int64_t floor_div(int64_t a, int64_t b) {
  int64_t q = a / b;
  if ((a % b != 0) && ((a < 0) != (b < 0))) --q;
  return q;
}

void or_fold_geometry(int64_t f, int64_t s, int64_t pw, int64_t KW,
                      int64_t* r, int64_t* c0, int64_t* kwf) {
  *r = f / s;
  *c0 = -ceil_div(pw, f);
  *kwf = floor_div(f - s - pw + KW - 1, f) - *c0 + 1;
}

void or_expand_filter_folded(const float* w, int64_t KH, int64_t KW, int64_t C,
                             int64_t Co, int64_t f, int64_t s, int64_t pw,
                             float* out) {
  int64_t r, c0, kwf;
  or_fold_geometry(f, s, pw, KW, &r, &c0, &kwf);
  const int64_t Cif = f * C, Cof = r * Co;
  memset(out, 0, (size_t)(KH * kwf * Cif * Cof) * sizeof(float));
  for (int64_t kh = 0; kh < KH; ++kh)
    for (int64_t kp = 0; kp < kwf; ++kp)
      for (int64_t fi = 0; fi < f; ++fi)
        for (int64_t j = 0; j < r; ++j) {
          const int64_t kw = (c0 + kp) * f + fi - j * s + pw;
          if (kw < 0 || kw >= KW) continue;
          for (int64_t c = 0; c < C; ++c)
            for (int64_t co = 0; co < Co; ++co)
              out[((kh * kwf + kp) * Cif + fi * C + c) * Cof + j * Co + co] =
                  w[((kh * KW + kw) * C + c) * Co + co];
        }
}

/* Folded conv evaluated the reference way: for every folded output pixel
 * (b, oh, w') and column (j, co), sum over (kh, kw', fi, c) in that order of
 * x_f * W' with out-of-range input (padding / beyond W) read as 0, into a
 * +0.0f float accumulator. Zero filter taps contribute exact +-0 products, so
 * on finite data this equals or_conv2d of the zero-padded input (SURVEY.md
 * Appendix A "Reduction order"). Writes the UNFOLDED output y (B,OH,OW,Co):
 * reconstruct_output is a reshape; columns ow >= OW (tail) are dropped. */
void or_conv_folded(const float* x, int64_t B, int64_t H, int64_t W, int64_t C,
                    const float* wexp, int64_t KH, int64_t KW, int64_t Co,
                    int64_t f, int64_t s, int64_t ph, int64_t pw, float* y) {
  int64_t r, c0, kwf;
  or_fold_geometry(f, s, pw, KW, &r, &c0, &kwf);
  const int64_t OH = (H + 2 * ph - KH) / s + 1, OW = (W + 2 * pw - KW) / s + 1;
  const int64_t Wfo = ceil_div(OW, r), Cif = f * C, Cof = r * Co;
  for (int64_t b = 0; b < B; ++b)
    for (int64_t oh = 0; oh < OH; ++oh)
      for (int64_t wp = 0; wp < Wfo; ++wp)
        for (int64_t n = 0; n < Cof; ++n) {
          const int64_t ow = wp * r + n / Co;
          if (ow >= OW) continue;
          float acc = 0.0f;
          for (int64_t kh = 0; kh < KH; ++kh) {
            const int64_t ih = oh * s - ph + kh;
            for (int64_t kp = 0; kp < kwf; ++kp)
              for (int64_t k = 0; k < Cif; ++k) {
                const int64_t iw = (wp + c0 + kp) * f + k / C;
                float xv = 0.0f;
                if (ih >= 0 && ih < H && iw >= 0 && iw < W)
                  xv = x[((b * H + ih) * W + iw) * C + k % C];
                acc += xv * wexp[((kh * kwf + kp) * Cif + k) * Cof + n];
              }
          }
          y[((b * OH + oh) * OW + ow) * Co + n % Co] = acc;
        }
}
