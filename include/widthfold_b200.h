/*
 * widthfold_b200.h -- C-ABI of the B200-native folded first-layer convolution.
 *
 * This is the drop-in boundary for the reference `widthfold` conv path. The
 * reference binds its path as free C++ functions in namespace widthfold
 * (no plugin registry): the entry points below replace them one-for-one.
 *
 *   wf_plan_fold            <- widthfold::check_legality / choose_fold_factor
 *                              /root/reference/proj/include/widthfold/fold.hpp:42-48
 *                              (src/fold.cpp:51-90), generalized to KW>1,
 *                              stride and padding.
 *   wf_packed_filter_bytes  <- (new) size of the once-per-weights packed filter.
 *   wf_expand_filter_pack   <- widthfold::expand_filter_general + replicate_bias
 *                              fold.hpp:71-74 (src/fold.cpp:185-226): the
 *                              block-structured expansion, written straight into
 *                              the tcgen05 shared-memory operand layout.
 *   wf_expand_filter_dense  <- widthfold::expand_filter_general, dense
 *                              (KH,KW',f*C,r*Cout) layout (bit-exact transform).
 *   wf_conv_fold_fwd        <- widthfold::conv2d + bias_add (+ReLU epilogue)
 *                              refconv.hpp:43-47 (src/refconv.cpp:34-95) on the
 *                              folded view, and reconstruct_output (a reshape:
 *                              the kernel writes final NHWC).
 *   wf_last_error           <- the message of the widthfold:: exception the C++
 *                              wrapper rethrows (include/widthfold/errors.hpp).
 *
 * Conventions: the caller owns every device buffer (no allocation inside
 * wf_conv_fold_fwd); calls are stream-ordered and asynchronous; plain
 * pointers and sizes only. Errors are status codes; wf_last_error() returns
 * a thread-local message for the last failing call on this thread.
 */
#ifndef WIDTHFOLD_B200_H_
#define WIDTHFOLD_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes map 1:1 onto the reference exception taxonomy
 * (include/widthfold/errors.hpp:11-52) plus std::invalid_argument. */
typedef enum {
  WF_OK = 0,
  WF_SHAPE_MISMATCH = 1,     /* widthfold::ShapeMismatch      errors.hpp:11  */
  WF_DEGENERATE_OUTPUT = 2,  /* widthfold::DegenerateOutput   errors.hpp:16  */
  WF_ILLEGAL_FOLD = 3,       /* widthfold::IllegalFold        errors.hpp:21  */
  WF_NOT_BLOCK_DIAGONAL = 4, /* widthfold::NotBlockDiagonal   errors.hpp:26  */
  WF_INVALID_ARGUMENT = 5,   /* std::invalid_argument (src/fold.cpp:44-47)   */
  WF_UNSUPPORTED = 6,        /* legal fold the sm_100a kernel cannot run     */
  WF_CUDA_ERROR = 7
} wf_status;

/* Arithmetic type the tensor cores consume. WF_TF32 = fp32 buffers,
 * kind::tf32 MMA; WF_F32 is accepted only as an output type. */
typedef enum { WF_F32 = 0, WF_TF32 = 1, WF_BF16 = 2, WF_F16 = 3 } wf_dtype;

/* FoldReason, same order/meaning as include/widthfold/fold.hpp:14-23, then
 * the two reasons the generalized device fold adds. */
typedef enum {
  WF_REASON_NONE = 0,
  WF_REASON_WIDTH_NOT_DIVISIBLE = 1,
  WF_REASON_KERNEL_SPANS_FOLD_AXIS = 2,
  WF_REASON_STRIDE_ON_FOLD_AXIS = 3,
  WF_REASON_ALREADY_ALIGNED = 4,
  WF_REASON_FACTOR_TOO_LARGE = 5,
  WF_REASON_UNSUPPORTED_CHANNELS = 6,
  WF_REASON_NOT_PROFITABLE = 7,
  WF_REASON_UNALIGNED_PIXEL = 8, /* f*C*elem not a multiple of the 32 B MMA K-step */
  WF_REASON_OUTPUT_TAIL = 9      /* reserved (OW % r != 0 is now a masked tail)     */
} wf_fold_reason;

typedef enum { WF_FOLD_APPLY = 0, WF_FOLD_FALLBACK = 1 } wf_fold_status;

/* Epilogue flags of wf_conv_fold_fwd[_ws]. WF_EPI_ROW_PRODUCER is a
 * cross-check, not a fast path: it builds the TMA-layout A tile with the
 * row-gather producer instead (same shared-memory image, bit-identical
 * output). Any other bit is rejected with WF_INVALID_ARGUMENT (profiling
 * switches exist only in a WFB_PROFILE=1 build of the library). */
typedef enum {
  WF_EPI_NONE = 0,
  WF_EPI_BIAS = 1,
  WF_EPI_RELU = 2,
  WF_EPI_PREPITCHED = 4,  /* the workspace already holds x re-pitched (wf_repitch_input): skip that pass */
  WF_EPI_ROW_PRODUCER = 0x4000
} wf_epilogue;

/* Kernel variant: the width-folded conv, or the same tcgen05 kernel on the
 * unfolded Cin=C input (explicit im2col A tiles) for the comparison. The
 * zero-padded Cin 3->8 variant is the folded kernel on a padded tensor. */
typedef enum { WF_VARIANT_FOLD = 0, WF_VARIANT_UNFOLDED = 1 } wf_variant;

/* Conv problem: x NHWC (n,h,w,c), w HWIO (kh,kw,c,cout), symmetric padding. */
typedef struct {
  int64_t n, h, w, c, kh, kw, cout, stride_h, stride_w, pad_h, pad_w;
} wf_conv_desc;

/* Result of planning. The first block mirrors widthfold::FoldPlan
 * (fold.hpp:28-37); the rest is the device schedule derived from it. */
typedef struct {
  int32_t status;          /* wf_fold_status */
  int32_t reason;          /* wf_fold_reason */
  int64_t f;               /* fold factor F */
  int64_t r;               /* outputs per folded column = f / stride */
  int64_t c0;              /* first folded column read, -ceil(pad_w / f) */
  int64_t kw_f;            /* KW' folded filter width */
  int64_t k_f;             /* dense folded K = KH*KW'*f*C */
  int64_t cout_f;          /* folded output channels = r*Cout */
  /* device schedule (valid when status == WF_FOLD_APPLY) */
  int32_t in_dtype;        /* wf_dtype the plan was made for */
  int32_t elem_bytes;      /* input element size */
  int64_t oh, ow;          /* output extent */
  int64_t wf, wfo;         /* folded input / output columns */
  int64_t units_per_px;    /* 32-byte MMA K-steps per folded pixel */
  int64_t group_size;      /* output sub-columns j per MMA group */
  int64_t n_groups;        /* r / group_size */
  int64_t n_tiles;         /* N-tiles (each <= 256 accumulator columns) */
  int64_t tile_rows;       /* output rows per M tile (OHt) */
  int64_t wbox;            /* folded columns loaded per output row (Wfo+KW'-1) */
  int64_t nrows;           /* input rows per residue region */
  int64_t mma_entries;     /* tcgen05.mma instructions per M tile (all N-tiles) */
  int64_t table_bytes;     /* schedule table size inside the packed buffer */
  int64_t packed_bytes;    /* = wf_packed_filter_bytes */
  int64_t epi_chunk;       /* accumulator columns per epilogue chunk: the period
                              of the output-column permutation baked into the
                              packed filter (coalesced 16x256b TMEM reads) */
  int32_t variant;         /* wf_variant */
  int32_t producer;        /* A-tile producer: 0 TMA boxes on x, 1 row gather
                              (folded layout), 2 row gather (explicit im2col),
                              3 re-pitch x into the workspace, then TMA boxes,
                              4 rows staged in shared memory + gather warps,
                              5 gather warps re-pitch each stage unit into a
                              ring in the workspace (L2-resident), then TMA
                              boxes, 6 gather warps load the rows straight from
                              x (L2-prefetched) into the A layout -- rows whose
                              pitch TMA cannot address */
  int32_t cta_pair;        /* 2: the conv runs on CTA pairs (cta_group::2, M = 256
                              per MMA), each SM holding half of every B block */
  int32_t stage_tiles;     /* M tiles fed by one A stage: 2 when two consecutive
                              output-row bands share their input-row halo */
  int32_t kstep_mode;      /* MMA K-steps: 0 32-byte covers of each kh row's
                              window, 1 cross-kh pairs of 16-byte core columns */
  int32_t launch_opts;     /* launch tuning decided at plan time (never read
                              from the environment at launch): bit 0 two TMEM
                              accumulator buffers only, bits 1-2 epilogue
                              ping-pong (0 default = off, 1 off, 2 on), bit 3
                              / bit 4 force the multicast N-tile cluster off /
                              on (plans with two N-tiles; default on only for
                              TMA boxes straight from x over >= 2 H-stride
                              residues) */
  int64_t pitched_w;       /* producers 3, 5: re-pitched row width (>= W, % f == 0) */
  int64_t workspace_bytes; /* device scratch wf_conv_fold_fwd_ws needs (0: none) */
  uint64_t useful_macs;    /* count_macs of the original conv */
  uint64_t issued_macs;    /* MACs the tensor cores execute (128-row tiles) */
} wf_fold_plan;

/* Plan a generalized width fold. f == 0 picks the factor automatically
 * (smallest f with f % stride == 0 and f*C*elem a multiple of 32 bytes);
 * group_size == 0 picks the MMA grouping. Legality failures come back as
 * status == WF_FOLD_FALLBACK with a reason, never as an error
 * (fold.hpp:39-41). Errors: WF_SHAPE_MISMATCH, WF_DEGENERATE_OUTPUT,
 * WF_INVALID_ARGUMENT. Host-only, pure, reentrant. */
wf_status wf_plan_fold(const wf_conv_desc* desc, int64_t f, int64_t group_size,
                       wf_dtype in_dtype, wf_fold_plan* plan);

/* Plan the UNFOLDED variant (M row = output pixel, explicit im2col, same
 * MMA/epilogue). bf16/f16 only; Cout a multiple of 32. */
wf_status wf_plan_unfolded(const wf_conv_desc* desc, wf_dtype in_dtype, wf_fold_plan* plan);

/* Bytes of the packed filter buffer (schedule table + packed B operand). */
size_t wf_packed_filter_bytes(const wf_fold_plan* plan);

/* Expand (generalized block-diagonal, Appendix A) and pack the filter once:
 * w (kh,kw,c,cout) in plan->in_dtype (fp32 for WF_TF32) on device,
 * b (cout) fp32 on device or NULL. Writes w_packed (wf_packed_filter_bytes)
 * and b_rep (r*cout fp32, replicate_bias) when b_rep != NULL. */
wf_status wf_expand_filter_pack(const void* w, const float* b,
                                const wf_conv_desc* desc,
                                const wf_fold_plan* plan, void* w_packed,
                                float* b_rep, void* stream);

/* Dense generalized expansion W'(KH,KW',f*C,r*Cout), fp32 in/out, on device.
 * At KW=1, stride=1, pad=0 it equals expand_filter_general bit-for-bit. */
wf_status wf_expand_filter_dense(const float* w, const wf_conv_desc* desc,
                                 int64_t f, float* w_dense, void* stream);

/* y = ReLU?(conv(x, w) + b?) in NHWC. x: (n,h,w,c) in plan->in_dtype,
 * y: (n,oh,ow,cout) in out_dtype (WF_F32, WF_BF16 or WF_F16).
 * epilogue: WF_EPI_* flags; WF_EPI_BIAS needs b_rep from wf_expand_filter_pack.
 * No allocations; asynchronous on `stream` (a cudaStream_t). The kernel is
 * launched with programmatic stream serialization: its prologue (barrier
 * init, TMEM allocation, the bulk copy of w_packed) may overlap the previous
 * kernel on the stream; every other global access (x, workspace, b_rep, y)
 * waits on griddepcontrol.wait, so stream order holds for them. w_packed is
 * read early because only wf_expand_filter_pack writes it: the first conv
 * launch after a pack (or a wf_replicate_bias) is made without the attribute.
 * Write w_packed any other way (a memcpy into the buffer) and synchronize the
 * stream before the next conv. The environment variable WF_PDL=0 at first use
 * of a plan/buffer set turns PDL off. */
wf_status wf_conv_fold_fwd(const void* x, const void* w_packed,
                           const float* b_rep, void* y,
                           const wf_conv_desc* desc, const wf_fold_plan* plan,
                           wf_dtype out_dtype, uint32_t epilogue, void* stream);

/* Same, with the caller-owned device workspace plan->workspace_bytes long
 * (rows whose pitch is not a 16-byte multiple, e.g. AlexNet's 227-pixel rows:
 * producer 5 re-pitches each stage unit into a ring of slots there inside the
 * kernel -- a few tens of MB, batch-independent; producer 3 re-pitches the
 * whole batch there first). wf_conv_fold_fwd is this call
 * with workspace == NULL and fails with WF_INVALID_ARGUMENT for such plans. */
wf_status wf_conv_fold_fwd_ws(const void* x, void* workspace, const void* w_packed, const float* b_rep, void* y,
                              const wf_conv_desc* desc, const wf_fold_plan* plan, wf_dtype out_dtype,
                              uint32_t epilogue, void* stream);

/* Exact-order fp32 direct convolution on CUDA cores: widthfold::conv2d
 * (src/refconv.cpp:34-80) bit-for-bit (kh -> kw -> ci, no FMA) plus explicit
 * zero padding. The reference-semantics path for shapes/precisions the folded
 * tcgen05 kernel does not cover, and the engine of grouped_conv. */
/* The re-pitch pass of a plan with a workspace (producer 3) on its own:
 * writes x into workspace exactly as wf_conv_fold_fwd_ws would before its conv.
 * With WF_EPI_PREPITCHED the conv then skips the pass, so a caller can
 * re-pitch the next chunk of a batch on a second stream while the current
 * chunk is convolved. No-op (WF_OK) unless the plan re-pitches its input
 * (plan->producer == 3); WF_EPI_PREPITCHED is ignored by other plans. */
wf_status wf_repitch_input(const void* x, void* workspace, const wf_conv_desc* desc, const wf_fold_plan* plan,
                           void* stream);

wf_status wf_conv_direct_fwd(const float* x, const float* w, float* y, const wf_conv_desc* desc, void* stream);

/* Grouped exact-order fp32 conv (widthfold::grouped_conv, src/blockdiag.cpp:138-187):
 * w_dense is the (kh,kw,c,cout) block-diagonal filter; output channel oc of
 * block g = oc / (cout/groups) sums only input channels of block g, in the
 * reference order -- bit-identical to wf_conv_direct_fwd on finite data, and
 * off-block terms are never formed (a NaN/Inf input poisons only its block).
 * Run wf_check_block_diagonal first to enforce the strict-zero structure. */
wf_status wf_conv_grouped_fwd(const float* x, const float* w_dense, float* y, const wf_conv_desc* desc,
                              int64_t groups, void* stream);

/* out = ReLU?(y + b[i % c]) -- widthfold::bias_add (src/refconv.cpp:82-95). */
wf_status wf_bias_add(const float* y, const float* b, float* out, int64_t n, int64_t c, int32_t relu, void* stream);

/* y = (bf16 | f16) x, round to nearest even: the device dtype of a graph node
 * the pass folds at bf16/f16 precision (the reference graph is f32). No
 * reference counterpart. */
wf_status wf_cast_f32(const float* x, void* y, int64_t n, wf_dtype to, void* stream);

/* out[j*cout + co] = b[co], j < r -- widthfold::replicate_bias (src/fold.cpp:213-226). */
wf_status wf_replicate_bias(const float* b, int64_t cout, int64_t r, float* out, void* stream);

/* Strict-zero block-diagonal check of a dense (kh,kw,cif,cof) fp32 filter for
 * `groups` blocks (src/blockdiag.cpp:24-84). scratch: 8 bytes of device
 * memory. *first_bad = flat index of the first offending entry or -1.
 * Synchronizes `stream`. Returns WF_NOT_BLOCK_DIAGONAL when one is found. */
wf_status wf_check_block_diagonal(const float* w_dense, int64_t kh, int64_t kw, int64_t cif, int64_t cof,
                                  int64_t groups, void* scratch, int64_t* first_bad, void* stream);

/* Diagnostic: the tcgen05 schedule make_schedule builds for (desc, f,
 * group_size, in_dtype) as one JSON object (A-stage layout, per-MMA
 * descriptor offsets, per-core-column (kh, c, slot mask) words, slot order) in
 * buf (cap bytes, NUL-terminated). Lets a host-side simulator replay the MMAs
 * against the oracle without a GPU. Host-only. WF_INVALID_ARGUMENT if cap is
 * too small or the plan falls back. No reference counterpart. */
wf_status wf_schedule_describe(const wf_conv_desc* desc, int64_t f, int64_t group_size, wf_dtype in_dtype,
                               char* buf, size_t cap);

/* Number of SMs the conv kernel assumes (persistent grid); 0 = device value. */
void wf_set_num_sms(int num_sms);

/* Thread-local message of the last failing call on this thread. */
const char* wf_last_error(void);

/* ABI version for the host wrappers. */
int wf_abi_version(void);

#ifdef __cplusplus
}
#endif

#endif /* WIDTHFOLD_B200_H_ */
