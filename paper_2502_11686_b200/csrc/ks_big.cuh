// Large-n path (ks_big.cu): batched dense building blocks and the level
// orchestration over HBM-resident block columns.
#pragma once
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <vector>

namespace ks {
namespace big {

extern std::atomic<int64_t> g_launches;   // kernels launched by this path (ks_info)
constexpr int kBigNB = 16;          // Householder panel width
constexpr int kBigMaxRows = 1600;   // rows of a stage stack (panel in shared memory)

// strided-batched C = alpha op(A) op(B) + beta C, column-major
struct Gemm {
  const double *A = nullptr, *B = nullptr;
  double *C = nullptr;
  int64_t sA = 0, sB = 0, sC = 0, batch = 1;
  int lda = 1, ldb = 1, ldc = 1, M = 0, N = 0, K = 0;
  double alpha = 1.0, beta = 0.0;
};
cudaError_t gemm(const Gemm &g, bool ta, bool tb, cudaStream_t s);

// batched block copy descriptor (see big_copy_kernel)
struct CopyDesc {
  const double *src = nullptr;   // null: zeros (plus diag on the diagonal)
  double *dst = nullptr;
  int64_t ss = 0, sd = 0, count = 0;
  int lds = 1, ldd = 1, rows = 0, cols = 0;
  double alpha = 1.0, diag = 0.0;
  int trans = 0, upper = 0;
};
constexpr int kMaxCopies = 12;
struct CopyList {
  CopyDesc d[kMaxCopies];
  int count = 0;
  void add(const CopyDesc &c) {
    if (c.count > 0 && c.rows > 0 && c.cols > 0) d[count++] = c;
  }
};
cudaError_t copy(const CopyList &L, int64_t batch, cudaStream_t s);

struct Panel {
  double *S;
  int64_t sS;
  int lds, m, j0, nb;
  double *V, *U;      // V written at V (explicit, rows x nb), U = V T^T at U
  int64_t sV, sU;
  int ldv, ldu;
  double *tau;        // tau_j at tau[j] (per item stride stau)
  int64_t stau;
};
constexpr int kBigBlk = 64;   // block reflector width of the trailing updates (4 panels)
// per-item QR scratch: V, U (rows x 64), U16 (rows x 16), W (64 x cols),
// G = V^T V and T (64 x 64), tau (64)
struct Work {
  double *V, *U, *U16, *W, *G, *T, *tau;
  int64_t sVU, sU16, sW, sGT, stau;
  int ldv;
  // lookahead (qr_apply): a second V / U pair (blocks alternate) and W for
  // the trailing update that runs on `side` while the next block's panels
  // run on the calling stream; side == null: no lookahead
  double *V2 = nullptr, *U2 = nullptr, *Wt = nullptr;
  cudaStream_t side = nullptr;
  cudaEvent_t evf = nullptr, evj = nullptr;
};
cudaError_t qr_apply(double *S, int64_t sS, int lds, int m, int ncols_fac, int ncols, int64_t batch,
                     const Work &w, cudaStream_t s);

struct Trsm {
  const double *R;
  int64_t sR;
  int ldr;
  double *B;
  int64_t sB;
  int ldb, k;
  int upper;
};
cudaError_t trsm(const Trsm &a, int n, int64_t batch, cudaStream_t s);
cudaError_t chol(double *A, int64_t sA, int ld, int d, int64_t batch, bool given, unsigned long long *status,
                 int64_t step_off, int64_t step_mul, int kind, cudaStream_t s);
cudaError_t sumsq(const double *A, int64_t sA, int lda, int rows, int cols, double *out, int64_t so, bool acc,
                  int64_t batch, cudaStream_t s);
cudaError_t rank_check(const double *R, int64_t sR, int ldr, int n, const double *nrm2, int64_t snrm,
                       unsigned long long *status, int64_t step_first, int64_t step_stride, int64_t batch,
                       cudaStream_t s);
cudaError_t sym_store(const double *A, int64_t sA, int lda, double *dst, int64_t sd, int n, int64_t batch,
                      cudaStream_t s);

// Everything the large-n orchestration needs (laid out by ks_api.cu's carve).
// Blocks are column-major; level >= 1 entries are AoS per column:
//   [C (n x n) | y (n) | El (n x n) | Er (n x n) | e (n) | |column|^2 (1)]
// records per eliminated column: [T_l (n x n) | T_r (n x n) | w (n) | P (n x n)]
// cross blocks per level: X[c] = S_{c, c-1} (n x n), c = 1 .. K-1.
struct Plan {
  int n = 0, RC = 0, mx = 0;
  int64_t N = 0, cntE = 1, cntC = 1, seg = 1;
  bool constC = true, chol = false;
  // inputs (device, ABI row-major blocks)
  const int32_t *m = nullptr;
  const double *F = nullptr, *H = nullptr, *c = nullptr, *o = nullptr, *K = nullptr, *L = nullptr;
  int64_t sF = 0, sH = 0, sc = 0, so = 0, sK = 0, sL = 0;
  // whitening scratch and level-0 blocks
  double *Kw = nullptr, *Bw = nullptr, *Lw = nullptr, *Hw = nullptr;
  double *C0 = nullptr, *y0 = nullptr, *El0 = nullptr, *Er0 = nullptr, *e0 = nullptr;
  double *nC = nullptr, *nEr = nullptr, *nEl = nullptr, *nrm0 = nullptr;
  // levels
  std::vector<int64_t> Ks;
  std::vector<double *> ent, rec, X;
  // stage / backward scratch
  double *S1 = nullptr, *S2 = nullptr, *S3 = nullptr, *Rinv = nullptr, *SII = nullptr, *G = nullptr,
         *Pt = nullptr, *xg = nullptr, *xt = nullptr;
  Work w{}, w2{};           // QR scratch of the main and the second stream
  cudaStream_t s2 = nullptr;  // second stream (stage 3 beside stage 2), null: serial
  cudaEvent_t ev[2] = {nullptr, nullptr};
  // outputs
  double *x = nullptr, *S = nullptr;
  unsigned long long *status = nullptr;
};
int64_t entry_doubles_big(int n);
int64_t rrec_doubles_big(int n);
// scratch sizes (doubles) for the plan's first level
void scratch_sizes(const Plan &p, int64_t &s1, int64_t &s2, int64_t &s3, int64_t &vu, int64_t &w, int64_t &items);
int64_t max_stack_rows(int n, int RC);
cudaError_t whiten(const Plan &p, cudaStream_t s);
cudaError_t factor(const Plan &p, cudaStream_t s);
cudaError_t backward(const Plan &p, bool do_state, bool do_cov, cudaStream_t s);

}  // namespace big
}  // namespace ks
