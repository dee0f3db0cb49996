// Internal declarations shared by the ks kernels and the host ABI.
// (Not shared with oracle/ -- the oracle has its own, independent C code.)
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace ks {

// Status word: min over (prio << 56) | (step+1) << 8 | kind, written with
// atomicMin.  Input errors (K, L not SPD, data outside the exponent range:
// prio 0) win over the rank failures they cause downstream (prio 1), then
// the smallest step.
enum BadKind : int { kBadK = 1, kBadL = 2, kBadRank = 3, kBadScale = 4 };
constexpr unsigned long long kStatusOk = ~0ull;
__host__ __device__ inline unsigned long long status_word(int64_t step, int kind) {
  return ((unsigned long long)(kind == kBadRank ? 1 : 0) << 56) | ((unsigned long long)(step + 1) << 8) |
         (unsigned long long)kind;
}
__host__ __device__ inline int64_t status_step(unsigned long long st) {
  return (int64_t)((st >> 8) & ((1ull << 48) - 1)) - 1;
}

// Relative rank tolerance: |R_jj[d][d]| <= 1e-12 * |block column j of UA|_F
// (the Frobenius norm of the original whitened block column, which Q^T
// preserves; reading R9).
constexpr double kRankTol = 1e-12;

// A level's reduced system: column t owns a C-like block
// C_t [RC x n] with RHS y_t [RC], and (if it has a left neighbour) the
// coupling row [El_t | Er_t] (n x n each, acting on columns t-1 and t) with
// RHS e_t.  Level 0: C = W G, El = -V F, Er = V, e = V c.
struct EntryView {
  const double *C, *y, *El, *Er, *e;
  int64_t sC, sy, sEl, sEr, se;  // per-column strides in doubles (0 = constant)
  const double *nrm;             // |UA block column|_F of the column (null at level 0:
  int64_t snrm;                  //  computed from the whitened blocks)
  int RC;                        // row capacity of C (zero padded)
};

// AoS layout of a level >= 1 entry:
//   [C (n x n) | y (n) | El (n x n) | Er (n x n) | e (n) | nrm (1)]
__host__ __device__ inline int64_t entry_doubles(int n) { return 3ll * n * n + 2ll * n + 1; }
// R record of an eliminated column: [Tl (n x n) | Tr (n x n) | P (n x n) | w (n)]
__host__ __device__ inline int64_t rrec_doubles(int n) { return 3ll * n * n + n; }

struct FactorLevelArgs {
  EntryView in;
  double *next;          // level L+1 entries, AoS, entry_doubles(n) each
  double *rrec;          // R records, rrec_doubles(n) each, index t/2
  int64_t K;             // columns at this level
  int64_t t0;            // global offset of column 0 (has_left(t) = t + t0 > 0)
  int n;
  int level;             // L: column t <-> step ((t + 1) << (level - lbase)) - 1 + step0
  int lbase;
  int64_t step0;         // for status reporting only
  unsigned long long *status;
  double *zscratch;      // n (n + 1) doubles: the odd level's last-column leftover Z (row-major)
                         // (+ one int flag behind it: split odd levels, set by launch_factor_level)
  int *zflag;            // null: the last pair's CTA also eliminates the last column
};

struct BackwardLevelArgs {
  const double *rrec;
  int64_t K, t0;
  int n;
  int shift;             // level - lbase: column t <-> domain index ((t + 1) << shift) - 1
  double *x;             // domain states   [*, n]
  double *S;             // domain covariances [*, n, n]
  const double *xhalo;   // domain index -1 (multi-GPU left neighbour), may be null
  const double *Shalo;
  const double *Xup;     // cross blocks of level L+1 (slot q at Xup + (q + 1) n^2), may be null
  double *Xcur;          // cross blocks of level L to write (null at level 0 / when not needed)
  int do_state, do_cov;
};

struct WhitenArgs {
  int64_t N;             // steps
  int n, m_max;
  const int32_t *m;      // [N] or null
  const double *F, *H, *c, *o, *K, *L;
  int64_t sF, sH, sc, so, sK, sL;
  int64_t first_global;  // global index of local step 0 (step 0 has no evolution row)
  // outputs
  double *C, *y, *El, *Er, *e;
  int64_t cntE, cntC;    // number of distinct evolution / observation blocks (1 or N)
  int constC;            // constant observation model (H, L stride 0, m = NULL): y by a separate kernel
  double *Mchol;         // [m_max x m_max] scratch when constC
  int chol;              // KS_COV_IS_CHOL: K, L already hold the lower Cholesky factors
  int64_t seg;           // steps per independent problem (global): step g has no evolution row iff g % seg == 0
  double *Mall;          // KS_KEEP_WHITENING: [cntC][m_max][m_max] lower factors M_i (row-major), or null
  // general model: evolution matrix H_i (null = I), rows l_i, state dims n_i (null: uniform)
  const double *Hev;
  int64_t sHev;
  const int32_t *l, *ns;
  int RC;                // rows of the whitened C blocks (m_max + padding rows e_k^T x_i = 0, k >= n_i)
  unsigned long long *status;
};

// ---------------------------------------------------------------------------
// Small-n path (n <= 8, m_max <= 8; ks_small.cu): one thread per column pair,
// blocks in registers, Givens row streaming, element-major (SoA) level arrays.
// ---------------------------------------------------------------------------
constexpr int kSmallMaxN = 8;
constexpr int kSmallMaxM = 8;

// Tiled ("AoSoA") view, 32 columns per tile: element e of column t lives at
//   p[(t >> 5) * ts + 32 e + (t & 31)]          (element stride ES = 32)
// so that a warp reading element e of 32 consecutive columns issues one
// coalesced 256-byte access and every element offset inside a column is a
// compile-time immediate; AoS records and constant blocks use
//   p[t * ts + e]                               (ES = 1; ts = 0: constant)
struct TView {
  double *p;
  int64_t ts;
};
__host__ __device__ inline int64_t tiled_doubles(int64_t cols, int64_t E) { return ((cols + 31) / 32) * 32 * E; }
// Pair-interleaved tiles (level-0 per-step arrays and level >= 1 entries of
// the small path): 64 columns per tile, even columns in the first half,
//   p[(t >> 6) * 64E + (t & 1) * 32E + 32 e + ((t >> 1) & 31)]
__host__ __device__ inline int64_t ptiled_doubles(int64_t cols, int64_t E) { return ((cols + 63) / 64) * 64 * E; }

struct SmallIn {               // level-L columns
  // level 0 (whitened inputs), one view per field (constant model: ES = 1,
  // ts = 0); C: RC x n row-major
  TView C, y, El, Er, e;
  TView nC, nEr, nEl;          // |C_j|^2, |Er_j|^2, |El_j|^2 (rank reference)
  int RC;
  // constant observation model: y = M^{-1} o computed by the level-0 factor
  // (yfuse = 1; Minv [RC][RC] lower triangular, o with stride so), else y
  int yfuse;
  const double *o, *Minv;
  int64_t so;
  // level >= 1: pair-interleaved tiled entry records [C (n x n, upper tri) | y | El | Er | e | nrm]
  TView ent;
};
struct SmallFactorArgs {
  SmallIn in;
  TView out;                   // level-(L+1) survivor entries: pair-interleaved tiled, or AoS (outAoS)
  TView rec;                   // tiled R records [Tl (n x n) | Tr (n x n) | w (n) | P (n(n+1)/2)]
  int64_t K, t0;
  int level, lbase;
  int64_t step0;
  unsigned long long *status;
  double *zscratch;            // n (n + 1) doubles: the odd level's last-column leftover Z
  int cE, cC, outAoS;          // level 0: constant evolution / observation blocks
  int64_t ent_off, out_off;    // fused kernels: entry / output column offsets of the CTA's buffers
};
// The fused recursion tail (small path): levels L_t .. top in one CTA.
constexpr int kMaxTailLevels = 16;
struct SmallTailArgs {
  SmallFactorArgs base;        // common fields (status, zscratch, t0 = 0, ...)
  const double *ent0;          // level-L_t entries (global, pair-interleaved tiles)
  int64_t W;                   // 0: one CTA, whole levels; else subtree width per CTA (power of 2)
  TView out_last;              // entries of the level after the last fused one (null at the top)
  int out_last_aos;            // out_last is an AoS entry (the sharded rank's boundary send buffer)
  int nlev;
  int64_t K[kMaxTailLevels];
  int level[kMaxTailLevels];
  TView rec[kMaxTailLevels];
};
struct SmallBackwardArgs {
  TView rec;                   // tiled R records
  int64_t K, t0;
  int shift;
  double *x, *S;               // domain outputs, row-major [*, n] / [*, n, n]
  const double *xhalo, *Shalo;
  TView Xup;                   // tiled S_{q,q+1} of level L+1 at column q+1 (p null: none)
  TView Xcur;                  // tiled level-L cross blocks to write (p null: skip)
  int do_state, do_cov;
};
// The backward of the fused tail: levels top .. L_t in one CTA (top first).
struct SmallBwdTailArgs {
  SmallBackwardArgs base;      // common fields (x, S, do_state, do_cov, t0 = 0, ...)
  int64_t W, nsub;             // 0: one CTA, whole levels; else subtree width (bottom level), CTAs
  int nlev;
  int64_t K[kMaxTailLevels];
  int shift[kMaxTailLevels];
  TView rec[kMaxTailLevels], Xup[kMaxTailLevels], Xcur[kMaxTailLevels];
};
struct SmallWhitenArgs {
  int64_t N;
  int n, m_max;
  const int32_t *m;
  const double *F, *H, *c, *o, *K, *L;
  int64_t sF, sH, sc, so, sK, sL;
  int64_t first_global;
  int64_t cntE, cntC;
  int constC;                  // constant observation model: y_i = M^{-1} o_i by small_whiten_y
  TView C, y, El, Er, e, nC, nEr, nEl;   // tiled per step, or ES = 1 / ts = 0 when constant
  int cE, cC;                  // layout flags of the above (1 = constant block)
  double *Mchol;               // m_max^2 scratch (constant observation model)
  double *Minv;                // m_max^2: M^{-1} for the factor's fused y (null: small_whiten_y)
  int chol;                    // KS_COV_IS_CHOL: K, L already hold the lower Cholesky factors
  int64_t seg;                 // steps per independent problem (global; see WhitenArgs)
  double *Mall;                // KS_KEEP_WHITENING: [cntC][m_max][m_max] lower factors M_i, or null
  const double *Hev;           // general model (see WhitenArgs)
  int64_t sHev;
  const int32_t *l, *ns;
  int RC;
  unsigned long long *status;
};
size_t small_entry_doubles(int n);                  // = entry_doubles(n)
int64_t small_rrec_doubles(int n);                  // 2 n^2 + n + n(n+1)/2
cudaError_t launch_small_whiten(const SmallWhitenArgs &a, cudaStream_t s, int *nlaunch);
cudaError_t launch_small_factor(const SmallFactorArgs &a, int n, cudaStream_t s);
cudaError_t launch_small_backward(const SmallBackwardArgs &a, int n, cudaStream_t s);
cudaError_t launch_small_factor_tail(const SmallTailArgs &t, int n, cudaStream_t s);
cudaError_t launch_small_backward_tail(const SmallBwdTailArgs &t, int n, cudaStream_t s);
int small_tail_max_cols(int n);     // levels with K <= this run in the fused tail kernel
// Multi-GPU boundary system on the small path: the P gathered AoS boundary
// entries (rank order) -> a pair-interleaved tiled level array of P columns.
cudaError_t launch_boundary_ptile(const double *recv, double *out, int P, int n, cudaStream_t s);
// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (kernel, device):
// the attribute belongs to a device context, so a per-process flag is wrong
// with several devices.  Thread-safe; kernels are identified by address.
cudaError_t set_smem_attr(const void *func, int bytes);
// cudaFuncAttributePreferredSharedMemoryCarveout = max shared, per (kernel, device)
cudaError_t set_carveout_max(const void *func);
// ks_update_obs: y_i = M_i^{-1} o_i (rows >= m_i zero) from the kept lower
// factors M (stride sM doubles per step: 0 = constant), written pair-
// interleaved tiled (small path, ptiled != 0) or row-major [N][m_max].
cudaError_t launch_update_y(const double *M, int64_t sM, const double *o, int64_t so, const int32_t *m, int mx,
                            int rc, int64_t N, double *y, int ptiled, cudaStream_t s);

// kernel launchers of the CTA path (ks_large.cu); return cudaGetLastError()
cudaError_t launch_whiten(const WhitenArgs &a, cudaStream_t s);
cudaError_t launch_factor_level(const FactorLevelArgs &a, cudaStream_t s);
cudaError_t launch_backward_level(const BackwardLevelArgs &a, cudaStream_t s);
size_t factor_smem_bytes(int n, int RC);
size_t backward_smem_bytes(int n);

}  // namespace ks
