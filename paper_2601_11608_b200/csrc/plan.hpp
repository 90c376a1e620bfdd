// plan.hpp -- generalized width-fold planner and tcgen05 schedule builder.
//
// Host-only, pure. Turns a conv problem (x NHWC, w HWIO, stride, padding) and
// a fold factor into (a) the FoldPlan facts the reference exposes
// (/root/reference/proj/include/widthfold/fold.hpp:28-37) and (b) the exact
// list of tcgen05.mma instructions one 128-row M tile issues.
//
// Geometry (the reference stops at KW == 1,
// src/fold.cpp:51-65):
//   r   = f / s                     output columns per folded column
//   c0  = -ceil(pw / f)             first folded column an output reads
//   KW' = floor((f-s-pw+KW-1)/f) - c0 + 1
//   folded output column w' covers ow = w'*r + j, j in [0, r); for input row
//   kh its window is the KW*C contiguous elements starting at element
//   off_j = (-c0*f + j*s - pw)*C of the KW'*f*C "window row".
//
// Shared-memory A operand (K-major, no swizzle, canonical 8x16 B core
// matrices): for each residue b = (kh - ph) mod s a region
//   [core column q in 0..2U)[input row i in 0..NR)[folded col w'' in 0..Wbox)[16 B]
// loaded by ONE 5-D TMA box (non-monotonic strides, probed on B200). The M row
// m = t*Wbox + w' of kh's operand is smem row ((a-amin_b)*Wbox + w' + kw'),
// so every (kh, kw') view is the same buffer at a 16-byte-aligned row shift
// (descriptor start address), i.e. each input byte is fetched once per tile.
//
// K is cut into 32-byte MMA K-steps ("units": 16 bf16/fp16 or 8 tf32) made of
// two 16-byte core columns; a unit may start at ANY core column c of the
// window row (pixel kp = c / Q, column q = c % Q, Q = f*C*elem/16). The pair
// (Q-1, Q) straddles into the next folded pixel: region Q of the A tile is a
// second TMA box holding core column 0 loaded one folded column further, so
// every pair is (region q, region q+1) at the same row shift. Output columns
// are split into groups of `group_size` sub-columns j; group g issues only the
// units its windows touch -- the tensor-core analogue of grouped_conv
// (src/blockdiag.cpp:138-187), which skips the structural zeros of the
// block-diagonal expansion.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "widthfold_b200.h"

namespace wfb {

constexpr int kTileM = 128;           // tcgen05 M (cta_group::1)
constexpr int kMaxAccCols = 256;      // accumulator columns per N-tile (x2 buffers)
constexpr int kMaxResidues = 8;
constexpr int kMaxNTiles = 16;
constexpr int kMaxEntries = 384;     // schedule entries per launch (the kernel's constant-bank table)
constexpr int kSmemLimit = 227 * 1024;
constexpr int kStagingBytes = 0;  // epilogue writes straight from registers (no staging)
constexpr int kRawSlots = 32;     // staged-row ring slots (row producer; >= the raw rows of a stage)
// L2 ring of re-pitched stage units (producer 5): slots per CTA and the CTA
// count the workspace is sized for (grids are <= the SM count: 148 on B200)
constexpr int kRingSlots = 3;
constexpr int kRingCtas = 160;
constexpr int kCtrlBytes = 2048;  // barriers, TMEM slot, row table at the base of shared memory
inline int raw_slot_bytes_for(int64_t row_bytes) { return static_cast<int>((row_bytes + 32 + 127) / 128 * 128); }

// Output-column permutation inside an epilogue chunk of CH accumulator
// columns. tcgen05.ld.16x256b hands thread t of a warp the columns
// 8i + 2(t%4) + {0,1} (i = 0..CH/8-1) of TMEM lanes t/4 and t/4+8; the packed
// filter puts output column (CH/4)*(t%4) + 2i + e of the chunk there, so each
// thread holds CH/4 CONSECUTIVE output channels and the 4 threads of a row
// cover CH contiguous channels: one full 128-byte line per row per store.
#ifdef __CUDACC__
#define WFB_HD __host__ __device__
#else
#define WFB_HD
#endif
WFB_HD inline int chunk_perm(int col, int CH) {
  const int c = col / CH, w = col % CH;
  return c * CH + (CH / 4) * ((w % 8) / 2) + 2 * (w / 8) + (w % 2);
}

struct MmaEntry {          // 16 bytes, lives in the packed buffer and in smem
  uint32_t a_off;          // byte offset of the A view inside an A stage
  uint32_t b_off;          // byte offset of the B block inside the N-tile's B
  uint32_t meta;           // kh | u << 8 | slot << 16 | (N/8) << 22 | accumulate << 31
                           // (kh, u: position of core column 0; slot: first accumulator slot)
  uint32_t tmem_col;       // accumulator column of the group
};

struct NTile {
  int g0, g1;              // groups [g0, g1)
  int col0, cols;          // output columns [col0, col0 + cols) of the r*Cout row
  int entry0, entries;     // slice of the schedule
  int split = -1;          // entries writing only the lower half of the columns
                           // (issued first; -1: no half-split of the accumulator)
  int64_t b_off, b_bytes;  // B region inside the packed buffer (after the table)
};

struct Schedule {
  wf_fold_plan plan{};
  int s = 1, ph = 0, pw = 0;
  int esize = 2;                 // input element bytes
  int E = 16;                    // elements per 32-byte unit
  int Q = 2;                     // 16-byte core columns per folded pixel
  bool need_shift = false;       // some unit pairs (Q-1, next pixel's 0)
  bool sw32 = false;             // A tile as SWIZZLE_32B regions of 32-byte K-steps
  std::vector<int> qs;           // sw32: in-pixel core-column offsets with a region each
  int qregion_bytes = 0;         // sw32: bytes of one such region (1024-aligned)
  int Ng = 64;                   // accumulator columns per group
  int CH = 64;                   // epilogue chunk (columns per 16x256b TMEM read)
  int prod = 0;                  // A producer: 0 TMA boxes, 1 row gather (folded), 2 row gather
                                 // (im2col), 3 re-pitch into the workspace + TMA boxes,
                                 // 4 rows staged in shared memory + gather warps,
                                 // 5 gather warps re-pitch each stage unit into an L2 ring + TMA boxes
  int64_t Wp = 0;                // input width the TMA view uses (re-pitched when != W)
  int pair = 1;                  // 2: CTA-pair (cta_group::2) MMAs, B blocks split across the pair
  int tps = 1;                   // M tiles per A stage (2: consecutive tiles share their input rows)
  int tile_shift = 0;            // bytes of A between the stage's tiles
  int U = 0;                     // im2col: 32-byte K-steps per kh
  int ksplit = 1;                // A stages per M tile (im2col: kh ranges)
  int raw_slots = 0, raw_slot_bytes = 0;  // staged-row ring of the row producer (prod 1/2)
  int ring_rows = 0;             // prod 5: input rows per ring slot (a stage unit's rows, re-pitched)
  int64_t ring_slot_bytes = 0;   // prod 5: bytes per ring slot (ring_rows x Wp*C*elem)
  int amin_min = 0;              // min over residues of amin (slot row 0 = input row (oh0 + amin_min) * s)
  std::vector<int> ks_kh0, ks_entry0, ks_entries, ks_chunks;
  int amin[kMaxResidues] = {0};
  int amax[kMaxResidues] = {0};
  bool has_res[kMaxResidues] = {false};
  int region_bytes = 0, stage_bytes = 0, lbo_a = 0;
  int stages = 2;
  int smem_bytes = 0, b_smem_bytes = 0, table_smem_bytes = 0;
  int64_t num_mtiles = 0, ohb = 0;
  std::vector<MmaEntry> entries;
  // Per entry, what each of its two 16-byte core columns holds:
  // kh | c << 8 | mask << 16 (c: core column of the KW'*f*C window row; mask:
  // the run's accumulator slots whose B rows are nonzero for it). Packed into
  // the header after the slot order; the pack kernel builds B from it.
  std::vector<uint32_t> entry_cc0, entry_cc1;
  std::vector<uint32_t> entry_lbo;  // per entry: A bytes from core column 0 to core column 1
  // Cross-kh core-column pairing: every MMA K-step is two single core columns
  // (8 bf16 / 4 tf32 elements) of any (kh, c) positions with the same output
  // groups -- K granularity 8 elements instead of 16 (no-swizzle A only).
  bool kpair = false;
  std::vector<NTile> ntiles;
  std::vector<int> order;        // accumulator slot (g0 + s of its N-tile) -> group
  std::vector<std::vector<int64_t>> units;  // per group: the first core columns of its K-steps
};

// Validates the descriptor like ConvSpec::validate (src/refconv.cpp:5-32) plus
// padding; throws nothing: returns a status and fills `err`.
wf_status validate_desc(const wf_conv_desc& d, std::string* err);

// Full planner. Returns WF_OK with plan.status == APPLY or FALLBACK (reason),
// or an error status (shape problems, bad arguments).
// kpair_req: -1 choose the K-step mode (cost model; WF_KPAIR=0/1 overrides),
// 0 / 1 force 32-byte covers / cross-kh core-column pairs. pair_req: -1 no CTA
// pairs unless WF_CTA_PAIR=1, 0 / 1 force. tps_req: -1 auto, 1 / 2 M tiles per A stage.
wf_status make_schedule(const wf_conv_desc& d, int64_t f, int64_t group_size,
                        wf_dtype in_dtype, Schedule* out, std::string* err, int kpair_req = -1,
                        int pair_req = -1, int tps_req = -1);

// The unfolded Cin=C variant of the same kernel (explicit im2col A tiles):
// the fold-vs-unfolded comparison of the north star.
wf_status make_schedule_unfolded(const wf_conv_desc& d, wf_dtype in_dtype, Schedule* out, std::string* err);

// Rebuild the schedule from a plan previously returned by make_schedule.
wf_status schedule_from_plan(const wf_conv_desc& d, const wf_fold_plan& p,
                             Schedule* out, std::string* err);

int elem_bytes(wf_dtype t);

}  // namespace wfb
