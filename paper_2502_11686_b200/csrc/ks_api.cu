// Host side of the C ABI declared in include/ks.h: argument checks, the
// workspace carve, the level plan (trailing-ones rule), the
// per-level launch loops, the multi-GPU boundary exchange and the status word.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nvtx3/nvToolsExt.h>

#include <cstdint>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <algorithm>
#include <new>
#include <vector>

#include "../../include/ks.h"
#include "ks_big.cuh"
#include "ks_internal.cuh"

using namespace ks;

namespace {

// NVTX range around every ABI phase (header-only NVTX v3: free without a
// profiler attached; nsys / ncu --nvtx show the phases of a step)
struct NvtxRange {
  explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

constexpr size_t kAlign = 256;
inline size_t align_up(size_t x) { return (x + kAlign - 1) & ~(kAlign - 1); }

struct Carve {
  char *base;
  size_t off = 0;
  template <class T>
  T *take(size_t count) {
    T *p = base ? reinterpret_cast<T *>(base + off) : nullptr;
    off = align_up(off + count * sizeof(T));
    return p;
  }
};

// ---- NCCL (dlopen'ed: the library has no link-time NCCL dependency) ----
struct NcclUid {
  char internal[128];
};
typedef int (*nccl_allgather_fn)(const void *, void *, size_t, int /*ncclDataType_t*/, void *,
                                 cudaStream_t);
typedef int (*nccl_uid_fn)(NcclUid *);
typedef int (*nccl_init_fn)(void **, int, NcclUid, int);
typedef int (*nccl_destroy_fn)(void *);
typedef int (*nccl_count_fn)(void *, int *);

struct Nccl {
  void *h = nullptr;
  nccl_allgather_fn allgather = nullptr;
  nccl_uid_fn uid = nullptr;
  nccl_init_fn init = nullptr;
  nccl_destroy_fn destroy = nullptr;
  nccl_count_fn count = nullptr;
  bool load() {
    if (h) return allgather && uid && init && destroy && count;
    // an NCCL already loaded into the process (PyTorch's) is found by its soname
    const char *names[] = {"libnccl.so.2", "libnccl.so"};
    for (const char *nm : names) {
      h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL);
      if (h) break;
    }
    if (!h) return false;
    allgather = (nccl_allgather_fn)dlsym(h, "ncclAllGather");
    uid = (nccl_uid_fn)dlsym(h, "ncclGetUniqueId");
    init = (nccl_init_fn)dlsym(h, "ncclCommInitRank");
    destroy = (nccl_destroy_fn)dlsym(h, "ncclCommDestroy");
    count = (nccl_count_fn)dlsym(h, "ncclCommCount");
    return allgather && uid && init && destroy && count;
  }
};
Nccl g_nccl;

}  // namespace

struct ks_dist {
  int rank = 0, nranks = 1;
  int64_t first = 0, nglobal = 0;
  void *comm = nullptr;   // ncclComm_t (library-owned) or null: caller-driven exchange
};

struct ks_ctx {
  ks_problem p{};
  int64_t N = 0;
  int n = 0, mx = 0;
  int rc = 0;             // rows of the whitened level-0 C blocks: m_max (+ n - nstate_min padding rows)
  bool general = false;   // the general model (Hev / l / nstate)
  cudaStream_t stream = nullptr;
  bool host_inputs = false;
  // sharding
  bool sharded = false;
  int rank = 0, nranks = 1, q = 0;
  void *comm = nullptr;   // the ks_dist's NCCL communicator (borrowed) or null
  // device views of the inputs
  const int32_t *m = nullptr, *l = nullptr, *ns = nullptr;
  const double *F = nullptr, *H = nullptr, *c = nullptr, *o = nullptr, *K = nullptr, *L = nullptr,
               *Hev = nullptr;
  // staging for host inputs
  int32_t *st_m = nullptr, *st_l = nullptr, *st_ns = nullptr;
  double *st_Hev = nullptr;
  size_t nHev = 0;
  double *st_F = nullptr, *st_H = nullptr, *st_c = nullptr, *st_o = nullptr, *st_K = nullptr,
         *st_L = nullptr;
  size_t nF = 0, nH = 0, nc = 0, no = 0, nK = 0, nL = 0;  // staged doubles
  // level 0 (whitened)
  unsigned long long *status = nullptr;
  double *C0 = nullptr, *y0 = nullptr, *El0 = nullptr, *Er0 = nullptr, *e0 = nullptr,
         *Mchol = nullptr, *Minv = nullptr;
  int64_t cntE = 1, cntC = 1;
  bool constC = true;     // constant observation model (H, L stride 0, m == NULL, uniform n_i)
  // local levels 0..nlev-1 (sharded: 0..q-1)
  std::vector<int64_t> K_;
  std::vector<double *> ent, rrec, X;
  // boundary levels (sharded)
  std::vector<int64_t> Kb;
  std::vector<double *> entb, rrecb, Xb;
  double *send = nullptr, *recv = nullptr, *bx = nullptr, *bS = nullptr, *hx = nullptr,
         *hS = nullptr, *Xq_local = nullptr;
  bool chol = false;      // KS_COV_IS_CHOL
  int64_t seg = 0;        // steps per independent problem (global steps; batch)
  double *Mall = nullptr; // KS_KEEP_WHITENING: per-step M_i
  // small-n path (ks_small.cu): element-major level arrays
  bool small = false;
  bool big = false;       // the large-n path (ks_big.cu): blocks beyond shared memory
  ks::big::Plan bp;
  double *nC0 = nullptr, *nEr0 = nullptr, *nEl0 = nullptr, *zscratch = nullptr;
  // outputs
  double *xout = nullptr, *Sout = nullptr;
  int stage = 0;  // 0 created, 1 whitened, 2 local-factored (sharded), 3 factored
  bool solved = false, covd = false;
  int64_t launches = 0;
  // timing
  bool timing = false;
  std::vector<cudaEvent_t> ev_pool;
  size_t ev_used = 0;
  std::vector<int> ev_family, ev_level;
  std::vector<int32_t> rec_family, rec_level;
  std::vector<float> rec_ms;
  double t_ms[KS_NFAMILIES] = {};
  int64_t t_cnt[KS_NFAMILIES] = {};
};

namespace {

int cuda_fail(cudaError_t e) {
  if (e == cudaSuccess) return KS_OK;
  fprintf(stderr, "[ks] CUDA error: %s\n", cudaGetErrorString(e));
  return KS_ERR_CUDA;
}

bool is_pow2(int64_t x) { return x > 0 && (x & (x - 1)) == 0; }

// Rows of the whitened level-0 C blocks: the observation rows, plus (per-step
// state dimensions n_i < n) the embedding's padding rows e_k^T x_i = 0 that
// pin the unused components k >= n_i of the uniform n-vector.
int level0_rows(const ks_problem *p) { return p->m_max + (p->nstate ? p->n - p->nstate_min : 0); }

bool use_small(const ks_problem *p) {
  return p->n <= kSmallMaxN && level0_rows(p) <= kSmallMaxM && !(p->flags & (KS_GENERIC_PATH | KS_BIG_PATH));
}

// The large-n path: blocks that do not fit the CTA path's shared memory
// (n = m = 500), or forced (KS_BIG_PATH, cross-checks).
bool use_big(const ks_problem *p) {
  if (use_small(p)) return false;
  if (p->flags & KS_BIG_PATH) return true;
  const int rc = level0_rows(p);
  return factor_smem_bytes(p->n, rc > p->n ? rc : p->n) > 227 * 1024 || backward_smem_bytes(p->n) > 227 * 1024;
}


constexpr uint32_t kAllFlags = KS_HOST_INPUTS | KS_OUTPUTS_BOUND | KS_GENERIC_PATH | KS_NO_FUSED_TAIL |
                               KS_COV_IS_CHOL | KS_KEEP_WHITENING | KS_BIG_PATH;

int64_t global_steps(const ks_problem *p, const ks_dist *d) { return (d && d->nranks > 1) ? d->nglobal : p->nsteps; }
int64_t segment_steps(const ks_problem *p, const ks_dist *d) {
  return global_steps(p, d) / (p->batch > 1 ? p->batch : 1);
}

int validate(const ks_problem *p, const ks_dist *d) {
  if (!p) return KS_ERR_ARG;
  if (p->nsteps < 1 || p->n < 1 || p->n > KS_MAX_N || p->m_max < 0 || p->m_max > KS_MAX_M)
    return KS_ERR_ARG;
  if (!p->F || !p->K || (p->m_max > 0 && (!p->H || !p->o || !p->L))) return KS_ERR_ARG;
  if (p->sF < 0 || p->sH < 0 || p->sc < 0 || p->so < 0 || p->sK < 0 || p->sL < 0) return KS_ERR_ARG;
  const int64_t n = p->n, mx = p->m_max;
  if ((p->sF && p->sF < n * n) || (p->sK && p->sK < n * n) || (p->sH && p->sH < mx * n) ||
      (p->sL && p->sL < mx * mx) || (p->sc && p->sc < n) || (p->so && p->so < mx))
    return KS_ERR_ARG;
  if (p->flags & ~kAllFlags) return KS_ERR_ARG;
  if (use_big(p)) {
    // one HBM-resident stage stack per pair; the Householder panel of a stack
    // (16 columns) must fit in shared memory; one GPU, uniform model
    if (ks::big::max_stack_rows(p->n, p->m_max) > ks::big::kBigMaxRows) return KS_ERR_ARG;
    if ((d && d->nranks > 1) || p->Hev || p->l || p->nstate || (p->flags & KS_KEEP_WHITENING)) return KS_ERR_ARG;
  }
  if (p->batch < 0 || (p->batch > 1 && global_steps(p, d) % p->batch != 0)) return KS_ERR_ARG;
  if (p->sHev < 0 || (p->sHev && p->sHev < n * n)) return KS_ERR_ARG;
  if (p->nstate && (p->nstate_min < 1 || p->nstate_min > p->n)) return KS_ERR_ARG;
  // per-step n_i on a shard: its first step's F_i is used unmasked (n_{i-1}
  // lives on the previous rank), so its columns >= n_{i-1} must be zero
  // (include/ks.h; dist.pad_shard zeroes them)
  if (d && d->nranks > 1) {
    // power-of-two shards in rank order (the local levels then follow the
    // global trailing-ones rule with no halo)
    if (!is_pow2(p->nsteps) || p->nsteps < 2) return KS_ERR_ARG;
    if (d->nglobal != p->nsteps * d->nranks || d->first != p->nsteps * d->rank) return KS_ERR_ARG;
  }
  return KS_OK;
}

// The level plan: level L has K_L columns,
// K_0 = N, K_{L+1} = floor(K_L / 2), down to one column (the base case,
// P:797-799); column t of level L is step ((t + 1) << L) - 1, the even
// columns (and an odd level's last column) are eliminated at L.  A sharded
// context stops before level `stop` (= log2 of its power-of-two shard).
std::vector<int64_t> level_sizes(int64_t N, int stop) {
  std::vector<int64_t> Ks;
  for (int64_t K = N, L = 0;; ++L) {
    if (L == stop) break;
    Ks.push_back(K);
    if (K == 1) break;
    K /= 2;
  }
  return Ks;
}

// Lay out (or just size, when base == nullptr) the workspace.
size_t carve(ks_ctx *c, char *base) {
  Carve w{base};
  const ks_problem &p = c->p;
  const int64_t N = c->N;
  const int n = c->n, mx = c->mx, rc = c->rc;
  const int64_t nn = (int64_t)n * n, E = entry_doubles(n), Rr = rrec_doubles(n);
  c->status = w.take<unsigned long long>(2);
  if (c->host_inputs) {
    auto cnt = [&](int64_t s, int64_t blk) { return (size_t)(s ? (N - 1) * s + blk : blk); };
    c->nF = cnt(p.sF, nn);
    c->nK = cnt(p.sK, nn);
    c->nH = mx ? cnt(p.sH, (int64_t)mx * n) : 0;
    c->nL = mx ? cnt(p.sL, (int64_t)mx * mx) : 0;
    c->no = mx ? cnt(p.so, mx) : 0;
    c->nc = p.c ? cnt(p.sc, n) : 0;
    c->st_m = p.m ? w.take<int32_t>(N) : nullptr;
    c->st_F = w.take<double>(c->nF);
    c->st_K = w.take<double>(c->nK);
    c->st_H = w.take<double>(c->nH);
    c->st_L = w.take<double>(c->nL);
    c->st_o = w.take<double>(c->no);
    c->st_c = p.c ? w.take<double>(c->nc) : nullptr;
    c->nHev = p.Hev ? cnt(p.sHev, nn) : 0;
    c->st_Hev = p.Hev ? w.take<double>(c->nHev) : nullptr;
    c->st_l = p.l ? w.take<int32_t>(N) : nullptr;
    c->st_ns = p.nstate ? w.take<int32_t>(N) : nullptr;
  }
  // a batch needs per-step evolution blocks (zero rows at every problem's first step)
  // (the general model: per-step unless only a constant H_i is given)
  c->cntE = (p.sF == 0 && p.sK == 0 && (p.c == nullptr || p.sc == 0) && p.batch <= 1 && p.sHev == 0 &&
             !p.l && !p.nstate) ? 1 : N;
  // constant observation model: one whitened C block, y = M^{-1} o from the one factor M
  c->constC = p.sH == 0 && p.sL == 0 && p.m == nullptr && !p.nstate;
  c->cntC = c->constC ? 1 : N;
  c->Mall = ((p.flags & KS_KEEP_WHITENING) && c->cntC > 1) ? w.take<double>(c->cntC * mx * mx + 1) : nullptr;
  const bool sm = c->small;
  const int64_t Rs = small_rrec_doubles(n);
  if (sm) {
    const bool cE = c->cntE == 1, cC = c->cntC == 1;
    auto sz = [&](bool cst, int64_t E) { return cst ? E : ptiled_doubles(N, E); };
    c->El0 = w.take<double>(sz(cE, nn));
    c->Er0 = w.take<double>(sz(cE, nn));
    c->e0 = w.take<double>(sz(cE, n));
    c->nEr0 = w.take<double>(sz(cE, 1));
    c->nEl0 = w.take<double>(sz(cE, 1));
    c->C0 = w.take<double>(sz(cC, (int64_t)rc * n) + 1);
    c->nC0 = w.take<double>(sz(cC, 1));
    c->y0 = w.take<double>(ptiled_doubles(N, rc) + 1);
    c->zscratch = w.take<double>(nn + n + 2);   // + the split-odd-level flag
  } else {
    c->El0 = w.take<double>(c->cntE * nn);
    c->Er0 = w.take<double>(c->cntE * nn);
    c->e0 = w.take<double>(c->cntE * n);
    c->C0 = w.take<double>(c->cntC * rc * n + 1);
    c->y0 = w.take<double>(N * rc + 1);
    c->zscratch = w.take<double>(nn + n + 2);   // + the split-odd-level flag
  }
  c->Mchol = w.take<double>((size_t)mx * mx + 1);
  c->Minv = w.take<double>((size_t)mx * mx + 1);
  // local levels
  c->K_ = level_sizes(N, c->sharded ? c->q : -1);
  c->ent.clear(); c->rrec.clear(); c->X.clear();
  for (size_t L = 0; L < c->K_.size(); ++L) {
    const int64_t K = c->K_[L];
    const int64_t ne = sm ? ptiled_doubles(K, E) : K * E;
    const int64_t nr = sm ? tiled_doubles((K + 1) / 2, Rs) : ((K + 1) / 2) * Rr;
    const int64_t nx = sm ? tiled_doubles(K + 1, nn) : (K + 1) * nn;
    c->ent.push_back(L == 0 ? nullptr : w.take<double>(ne));
    c->rrec.push_back(w.take<double>(nr));
    c->X.push_back(L == 0 ? nullptr : w.take<double>(nx));
  }
  if (c->big) {   // the large-n path's whitening and stage scratch (ks_big.cuh Plan)
    ks::big::Plan &b = c->bp;
    b.n = n; b.RC = rc; b.mx = mx; b.N = N; b.cntE = c->cntE; b.cntC = c->cntC;
    b.constC = c->constC; b.chol = c->chol; b.seg = c->seg;
    b.C0 = c->C0; b.y0 = c->y0; b.El0 = c->El0; b.Er0 = c->Er0; b.e0 = c->e0;
    b.Ks = c->K_; b.ent = c->ent; b.rec = c->rrec; b.X = c->X;
    b.Kw = w.take<double>(c->cntE * nn);
    b.Bw = w.take<double>(c->cntE * nn * 2 + c->cntE * n);
    b.Lw = w.take<double>(c->cntC * mx * mx + 1);
    b.Hw = w.take<double>(c->cntC * mx * (n + 1) + 1);
    b.nC = w.take<double>(c->cntC);
    b.nEr = w.take<double>(c->cntE);
    b.nEl = w.take<double>(c->cntE);
    b.nrm0 = w.take<double>(N);
    int64_t s1, s2, s3, vu, ww, items;
    ks::big::scratch_sizes(b, s1, s2, s3, vu, ww, items);
    b.S1 = w.take<double>(items * s1);
    b.S2 = w.take<double>(items * s2);
    b.S3 = w.take<double>(items * s3);
    const int64_t rows = vu / ks::big::kBigBlk;
    for (ks::big::Work *wk : {&b.w, &b.w2}) {   // one QR scratch per stream
      wk->V = w.take<double>(items * vu);
      wk->U = w.take<double>(items * vu);
      wk->V2 = w.take<double>(items * vu);       // lookahead: the alternate block's V, U
      wk->U2 = w.take<double>(items * vu);
      wk->Wt = w.take<double>(items * ww);
      wk->U16 = w.take<double>(items * rows * ks::big::kBigNB);
      wk->W = w.take<double>(items * ww);
      wk->G = w.take<double>(items * ks::big::kBigBlk * ks::big::kBigBlk);
      wk->T = w.take<double>(items * ks::big::kBigBlk * ks::big::kBigBlk);
      wk->tau = w.take<double>(items * ks::big::kBigBlk);
      wk->sVU = vu; wk->sU16 = rows * ks::big::kBigNB; wk->sW = ww;
      wk->sGT = ks::big::kBigBlk * ks::big::kBigBlk; wk->stau = ks::big::kBigBlk; wk->ldv = (int)rows;
    }
    b.Rinv = w.take<double>(items * nn);
    b.SII = w.take<double>(items * 4 * nn);
    b.G = w.take<double>(items * 2 * nn);
    b.Pt = w.take<double>(items * nn);
    b.xg = w.take<double>(items * 2 * n);
    b.xt = w.take<double>(items * n);
  }
  if (c->sharded) {
    const int P = c->nranks;
    c->send = w.take<double>(E);
    c->recv = w.take<double>((int64_t)P * E);
    c->Xq_local = w.take<double>(sm ? tiled_doubles(2, nn) : 2 * nn);
    c->hx = w.take<double>(n);
    c->hS = w.take<double>(nn);
    c->bx = w.take<double>((int64_t)P * n);
    c->bS = w.take<double>((int64_t)P * nn);
    c->Kb.clear(); c->entb.clear(); c->rrecb.clear(); c->Xb.clear();
    int64_t Kb = P;
    for (int L = 0;; ++L) {
      c->Kb.push_back(Kb);
      if (sm) {   // the boundary system runs on the small-path kernels (tiled level arrays)
        c->entb.push_back(w.take<double>(ptiled_doubles(Kb, E)));
        c->rrecb.push_back(w.take<double>(tiled_doubles((Kb + 1) / 2, Rs)));
        c->Xb.push_back(w.take<double>(tiled_doubles(Kb + 1, nn)));
      } else {    // generic AoS kernels
        c->entb.push_back(L == 0 ? c->recv : w.take<double>(Kb * E));
        c->rrecb.push_back(w.take<double>(((Kb + 1) / 2) * Rr));
        c->Xb.push_back(w.take<double>((Kb + 1) * nn));
      }
      if (Kb == 1) break;
      Kb /= 2;
    }
  }
  if (!(p.flags & KS_OUTPUTS_BOUND)) {
    c->xout = c->xout ? c->xout : w.take<double>(N * n);
    c->Sout = c->Sout ? c->Sout : w.take<double>(N * nn);
  }
  return w.off;
}

struct Launch {
  ks_ctx *c;
  int fam;
  cudaEvent_t e1 = nullptr;
  Launch(ks_ctx *c_, int f, int level, int nkernels = 1) : c(c_), fam(f) {
    if (c->timing) {
      if (c->ev_used + 2 > c->ev_pool.size()) {
        for (int i = 0; i < 64; ++i) {
          cudaEvent_t e;
          cudaEventCreate(&e);
          c->ev_pool.push_back(e);
        }
      }
      cudaEvent_t e0 = c->ev_pool[c->ev_used++];
      e1 = c->ev_pool[c->ev_used++];
      c->ev_family.push_back(f);
      c->ev_level.push_back(level);
      cudaEventRecord(e0, c->stream);
    }
    c->launches += nkernels;
  }
  ~Launch() {
    if (e1) cudaEventRecord(e1, c->stream);
  }
};

EntryView level0_view(const ks_ctx *c) {
  EntryView v;
  const int n = c->n, rc = c->rc;
  const int64_t nn = (int64_t)n * n;
  v.C = c->C0; v.sC = c->cntC == 1 ? 0 : (int64_t)rc * n;
  v.y = c->y0; v.sy = rc;
  v.El = c->El0; v.sEl = c->cntE == 1 ? 0 : nn;
  v.Er = c->Er0; v.sEr = c->cntE == 1 ? 0 : nn;
  v.e = c->e0; v.se = c->cntE == 1 ? 0 : n;
  v.nrm = nullptr; v.snrm = 0;
  v.RC = rc;
  return v;
}

EntryView aos_view(const double *ent, int n) {
  EntryView v;
  const int64_t E = entry_doubles(n), nn = (int64_t)n * n;
  v.C = ent; v.y = ent + nn; v.El = ent + nn + n; v.Er = ent + 2 * nn + n; v.e = ent + 3 * nn + n;
  v.nrm = ent + 3 * nn + 2 * n;
  v.sC = v.sy = v.sEl = v.sEr = v.se = v.snrm = E;
  v.RC = n;
  return v;
}

// ---- small-path views (tiled, 32 columns per tile; see TView) ----
TView tv(const double *p, int64_t ts) { return TView{const_cast<double *>(p), ts}; }

// Constant observation model on the small path: the level-0 factor computes
// y = M^{-1} o itself (no y pass over HBM).
int small_yfuse(const ks_ctx *c) {
  return (c->mx > 0 && c->constC) ? 1 : 0;
}

SmallIn small_level0(const ks_ctx *c) {
  const int n = c->n, rc = c->rc;
  const int64_t nn = (int64_t)n * n;
  const bool cE = c->cntE == 1, cC = c->cntC == 1;
  SmallIn v;
  v.C = tv(c->C0, cC ? 0 : 64 * (int64_t)rc * n);
  v.y = tv(c->y0, 64 * (int64_t)rc);
  v.El = tv(c->El0, cE ? 0 : 64 * nn);
  v.Er = tv(c->Er0, cE ? 0 : 64 * nn);
  v.e = tv(c->e0, cE ? 0 : 64 * (int64_t)n);
  v.nC = tv(c->nC0, cC ? 0 : 64);
  v.nEr = tv(c->nEr0, cE ? 0 : 64);
  v.nEl = tv(c->nEl0, cE ? 0 : 64);
  v.RC = rc;
  v.ent = tv(nullptr, 0);
  v.yfuse = small_yfuse(c);
  v.o = c->o;
  v.so = c->p.so;
  v.Minv = c->Minv;
  return v;
}

// One recursion on the small path: the local domain (levels 0..), or, on a
// sharded context, the P-column boundary system (global levels q..) that
// every rank factors redundantly with the same per-column routines (so the
// multi-GPU elimination order and arithmetic are the single-GPU ones).
struct SmallPlan {
  const std::vector<int64_t> *K;
  const std::vector<double *> *ent, *rrec, *X;
  bool l0;               // plan level 0 reads the whitened level-0 inputs
  bool local;            // the local domain (t0 = rank * K; subtree pass allowed)
  int lbase;             // global level of plan level 0 (status: plan-domain index)
  double *send;          // AoS output of the last level (sharded local domain), else null
  double *x, *S;         // plan-domain outputs
  const double *xhalo, *Shalo;
  double *Xtop;          // tiled cross blocks above the top level (sharded local: Xq_local)
  bool xcur0;            // write the level-0 cross blocks (boundary: scattered to the ranks)
};

SmallPlan local_plan(ks_ctx *c) {
  SmallPlan p;
  p.K = &c->K_; p.ent = &c->ent; p.rrec = &c->rrec; p.X = &c->X;
  p.l0 = true; p.local = true; p.lbase = 0;
  p.send = c->sharded ? c->send : nullptr;
  p.x = c->xout; p.S = c->Sout; p.xhalo = c->hx; p.Shalo = c->hS;
  p.Xtop = c->sharded ? c->Xq_local : nullptr;
  p.xcur0 = false;
  return p;
}

SmallPlan boundary_plan(ks_ctx *c) {
  SmallPlan p;
  p.K = &c->Kb; p.ent = &c->entb; p.rrec = &c->rrecb; p.X = &c->Xb;
  p.l0 = false; p.local = false; p.lbase = c->q;
  p.send = nullptr;
  p.x = c->bx; p.S = c->bS; p.xhalo = nullptr; p.Shalo = nullptr;
  p.Xtop = nullptr;
  p.xcur0 = true;
  return p;
}

SmallFactorArgs small_factor_args(ks_ctx *c, const SmallPlan &pl, size_t i) {
  const int n = c->n;
  const int64_t E = entry_doubles(n), Rs = small_rrec_doubles(n);
  const std::vector<int64_t> &Ks = *pl.K;
  SmallFactorArgs a;
  const bool last = i + 1 == Ks.size();
  a.in = small_level0(c);
  if (i > 0 || !pl.l0) a.in.ent = tv((*pl.ent)[i], 64 * E);
  a.outAoS = 0;
  if (!last) a.out = tv((*pl.ent)[i + 1], 64 * E);
  else if (pl.send) { a.out = tv(pl.send, E); a.outAoS = 1; }
  else a.out = tv(nullptr, 0);
  a.rec = tv((*pl.rrec)[i], 32 * Rs);
  a.t0 = (pl.local && c->sharded) ? (int64_t)c->rank * Ks[i] : 0;
  a.K = Ks[i];
  a.level = pl.lbase + (int)i;
  a.lbase = pl.lbase;
  a.step0 = 0;
  a.status = c->status;
  a.zscratch = c->zscratch;
  a.cE = c->cntE == 1;
  a.cC = c->cntC == 1;
  a.ent_off = a.out_off = 0;
  return a;
}

// First level run by the fused tail kernel (levels reading entries, with K
// <= the kernel's shared-memory capacity), or Ks.size() for none.
size_t small_tail_start(const ks_ctx *c, const SmallPlan &pl) {
  const std::vector<int64_t> &Ks = *pl.K;
  const int64_t cap = small_tail_max_cols(c->n);
  if (cap <= 0 || (c->p.flags & KS_NO_FUSED_TAIL)) return Ks.size();
  for (size_t i = pl.l0 ? 1 : 0; i < Ks.size(); ++i)
    if (Ks[i] <= cap) return (Ks.size() - i > (size_t)kMaxTailLevels) ? Ks.size() : i;
  return Ks.size();
}

// Subtree pass (levels [is, is + kSubLevels)): the first level ≥ 1 below the
// tail whose K is a multiple of the subtree width with at most one subtree
// per SM (the subtree kernel needs most of an SM's shared memory), local
// domain only; returns Ks.size() for none.
constexpr int kSubLevels = 7;   // subtree width 2^7 = 128 columns (tail_max_cols)
size_t small_subtree_start(const ks_ctx *c, const SmallPlan &pl) {
  const std::vector<int64_t> &Ks = *pl.K;
  const size_t it = small_tail_start(c, pl);
  const int64_t W = 1ll << kSubLevels;
  if (!pl.l0 || it >= Ks.size() || small_tail_max_cols(c->n) < W) return Ks.size();
  int dev = 0, sms = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  for (size_t i = 1; i + kSubLevels <= it; ++i)
    if (Ks[i] % W == 0 && Ks[i] / W <= sms) return i;   // one wave (one subtree per SM)
  return Ks.size();
}

SmallTailArgs small_tail_args(ks_ctx *c, const SmallPlan &pl, size_t i0, int nlev, int64_t W) {
  SmallTailArgs t;
  t.base = small_factor_args(c, pl, i0);
  t.ent0 = (*pl.ent)[i0];
  t.W = W;
  t.nlev = nlev;
  for (int l = 0; l < nlev; ++l) {
    t.K[l] = (*pl.K)[i0 + l];
    t.level[l] = pl.lbase + (int)(i0 + l);
    t.rec[l] = small_factor_args(c, pl, i0 + l).rec;
  }
  const SmallFactorArgs la = small_factor_args(c, pl, i0 + nlev - 1);
  t.out_last = la.out;
  t.out_last_aos = la.outAoS;
  return t;
}

int run_small_factor_levels(ks_ctx *c, const SmallPlan &pl, int fam) {
  const int n = c->n;
  const std::vector<int64_t> &Ks = *pl.K;
  const size_t it = small_tail_start(c, pl), is = small_subtree_start(c, pl);
  for (size_t i = 0; i < it;) {
    if (i == is) {   // kSubLevels levels in one launch, one subtree per CTA
      SmallTailArgs t = small_tail_args(c, pl, i, kSubLevels, 1ll << kSubLevels);
      Launch l(c, fam, pl.lbase + (int)i, 1);
      cudaError_t e = launch_small_factor_tail(t, n, c->stream);
      if (e != cudaSuccess) return cuda_fail(e);
      i += kSubLevels;
      continue;
    }
    SmallFactorArgs a = small_factor_args(c, pl, i);
    Launch l(c, fam, pl.lbase + (int)i);
    cudaError_t e = launch_small_factor(a, n, c->stream);
    if (e != cudaSuccess) return cuda_fail(e);
    ++i;
  }
  if (it < Ks.size()) {
    SmallTailArgs t = small_tail_args(c, pl, it, (int)(Ks.size() - it), 0);
    Launch l(c, fam, pl.lbase + (int)it, 1);
    cudaError_t e = launch_small_factor_tail(t, n, c->stream);
    if (e != cudaSuccess) return cuda_fail(e);
  }
  return KS_OK;
}

SmallBackwardArgs small_backward_args(ks_ctx *c, const SmallPlan &pl, int i, int do_state, int do_cov) {
  const int n = c->n;
  const int64_t nn = (int64_t)n * n, Rs = small_rrec_doubles(n);
  const std::vector<int64_t> &Ks = *pl.K;
  SmallBackwardArgs a;
  a.rec = tv((*pl.rrec)[i], 32 * Rs);
  a.K = Ks[i];
  a.shift = i;
  a.do_state = do_state;
  a.do_cov = do_cov;
  const bool top = i + 1 == (int)Ks.size();
  a.t0 = (pl.local && c->sharded) ? (int64_t)c->rank * Ks[i] : 0;
  a.x = pl.x; a.S = pl.S; a.xhalo = pl.xhalo; a.Shalo = pl.Shalo;
  if (!top) a.Xup = tv((*pl.X)[i + 1], 32 * nn);
  else a.Xup = tv(pl.Xtop, pl.Xtop ? 32 * nn : 0);
  a.Xcur = ((i >= 1 || pl.xcur0) && do_cov) ? tv((*pl.X)[i], 32 * nn) : tv(nullptr, 0);
  return a;
}

SmallBwdTailArgs small_bwd_tail_args(ks_ctx *c, const SmallPlan &pl, int top, int bottom, int do_state,
                                     int do_cov, int64_t W) {
  SmallBwdTailArgs t;
  t.base = small_backward_args(c, pl, top, do_state, do_cov);
  t.W = W;
  t.nsub = W ? (*pl.K)[bottom] / W : 1;
  t.nlev = 0;
  for (int i = top; i >= bottom; --i) {
    const SmallBackwardArgs a = small_backward_args(c, pl, i, do_state, do_cov);
    t.K[t.nlev] = a.K;
    t.shift[t.nlev] = a.shift;
    t.rec[t.nlev] = a.rec;
    t.Xup[t.nlev] = a.Xup;
    t.Xcur[t.nlev] = a.Xcur;
    ++t.nlev;
  }
  return t;
}

int run_small_backward_levels(ks_ctx *c, const SmallPlan &pl, int do_state, int do_cov, int fam) {
  const int n = c->n;
  const std::vector<int64_t> &Ks = *pl.K;
  const int it = (int)small_tail_start(c, pl);   // the levels the fused factor tail ran
  const int is = (int)small_subtree_start(c, pl);
  int top = (int)Ks.size() - 1;
  if (it < (int)Ks.size()) {
    SmallBwdTailArgs t = small_bwd_tail_args(c, pl, top, it, do_state, do_cov, 0);
    Launch l(c, fam, pl.lbase + it);
    cudaError_t e = launch_small_backward_tail(t, n, c->stream);
    if (e != cudaSuccess) return cuda_fail(e);
    top = it - 1;
  }
  for (int i = top; i >= 0;) {
    if (is < (int)Ks.size() && i == is + kSubLevels - 1) {   // the subtree pass, one subtree per CTA
      SmallBwdTailArgs t = small_bwd_tail_args(c, pl, i, is, do_state, do_cov, 1ll << kSubLevels);
      Launch l(c, fam, pl.lbase + is);
      cudaError_t e = launch_small_backward_tail(t, n, c->stream);
      if (e != cudaSuccess) return cuda_fail(e);
      i = is - 1;
      continue;
    }
    SmallBackwardArgs a = small_backward_args(c, pl, i, do_state, do_cov);
    Launch l(c, fam, pl.lbase + i);
    cudaError_t e = launch_small_backward(a, n, c->stream);
    if (e != cudaSuccess) return cuda_fail(e);
    --i;
  }
  return KS_OK;
}

int run_factor_levels(ks_ctx *c, bool boundary) {
  if (c->small) {
    if (!boundary) return run_small_factor_levels(c, local_plan(c), 1);
    // the gathered AoS boundary entries -> the plan's tiled level-0 array
    {
      Launch l(c, 4, c->q);
      cudaError_t e = launch_boundary_ptile(c->recv, c->entb[0], c->nranks, c->n, c->stream);
      if (e != cudaSuccess) return cuda_fail(e);
    }
    return run_small_factor_levels(c, boundary_plan(c), 4);
  }
  const int n = c->n;
  const std::vector<int64_t> &Ks = boundary ? c->Kb : c->K_;
  const int Lb = boundary ? c->q : 0;
  for (size_t i = 0; i < Ks.size(); ++i) {
    FactorLevelArgs a;
    const int L = Lb + (int)i;
    if (!boundary && i == 0) {
      a.in = level0_view(c);
    } else {
      a.in = aos_view(boundary ? c->entb[i] : c->ent[i], n);
    }
    a.K = Ks[i];
    a.n = n;
    a.level = L;
    a.lbase = boundary ? c->q : 0;
    a.status = c->status;
    a.zscratch = c->zscratch;
    if (boundary) {
      a.t0 = 0;
      a.step0 = 0;  // reported as boundary-domain index
      a.next = (i + 1 < Ks.size()) ? c->entb[i + 1] : nullptr;
      a.rrec = c->rrecb[i];
    } else {
      a.t0 = c->sharded ? (int64_t)c->rank * Ks[i] : 0;
      a.step0 = 0;
      if (i + 1 < Ks.size()) a.next = c->ent[i + 1];
      else a.next = c->sharded ? c->send : nullptr;
      a.rrec = c->rrec[i];
    }
    Launch l(c, boundary ? 4 : 1, L);
    cudaError_t e = launch_factor_level(a, c->stream);
    if (e != cudaSuccess) return cuda_fail(e);
  }
  return KS_OK;
}

// Timing families: 0 whiten, 1 factor levels, 2 solve levels, 3 selinv levels,
// 4 boundary system (multi-GPU), 5 fused solve+selinv levels.
int run_backward_levels(ks_ctx *c, bool boundary, int do_state, int do_cov) {
  if (c->small)
    return run_small_backward_levels(c, boundary ? boundary_plan(c) : local_plan(c), do_state, do_cov,
                                     boundary ? 4 : (do_cov ? (do_state ? 5 : 3) : 2));
  const int n = c->n;
  const std::vector<int64_t> &Ks = boundary ? c->Kb : c->K_;
  for (int i = (int)Ks.size() - 1; i >= 0; --i) {
    BackwardLevelArgs a;
    a.K = Ks[i];
    a.n = n;
    a.shift = i;
    a.do_state = do_state;
    a.do_cov = do_cov;
    if (boundary) {
      a.rrec = c->rrecb[i];
      a.t0 = 0;
      a.x = c->bx;
      a.S = c->bS;
      a.xhalo = nullptr;
      a.Shalo = nullptr;
      a.Xup = (i + 1 < (int)Ks.size()) ? c->Xb[i + 1] : nullptr;
      a.Xcur = c->Xb[i];
    } else {
      a.rrec = c->rrec[i];
      a.t0 = c->sharded ? (int64_t)c->rank * Ks[i] : 0;
      a.x = c->xout;
      a.S = c->Sout;
      a.xhalo = c->hx;
      a.Shalo = c->hS;
      if (i + 1 < (int)Ks.size()) a.Xup = c->X[i + 1];
      else a.Xup = c->sharded ? c->Xq_local : nullptr;
      a.Xcur = (i >= 1) ? c->X[i] : nullptr;
    }
    Launch l(c, boundary ? 4 : (do_cov ? (do_state ? 5 : 3) : 2), (boundary ? c->q : 0) + i);
    cudaError_t e = launch_backward_level(a, c->stream);
    if (e != cudaSuccess) return cuda_fail(e);
  }
  return KS_OK;
}

// Boundary results -> this rank's local domain (SURVEY §8(e) back phase).
int scatter_boundary(ks_ctx *c, bool states, bool cov) {
  const int n = c->n, r = c->rank;
  const int64_t nn = (int64_t)n * n, M = c->N;
  cudaError_t e = cudaSuccess;
  if (states) {
    e = cudaMemcpyAsync(c->xout + (M - 1) * n, c->bx + (int64_t)r * n, n * 8, cudaMemcpyDeviceToDevice, c->stream);
    if (r > 0 && e == cudaSuccess)
      e = cudaMemcpyAsync(c->hx, c->bx + (int64_t)(r - 1) * n, n * 8, cudaMemcpyDeviceToDevice, c->stream);
  }
  if (cov && e == cudaSuccess) {
    e = cudaMemcpyAsync(c->Sout + (M - 1) * nn, c->bS + r * nn, nn * 8, cudaMemcpyDeviceToDevice, c->stream);
    if (r > 0 && e == cudaSuccess) {
      e = cudaMemcpyAsync(c->hS, c->bS + (r - 1) * nn, nn * 8, cudaMemcpyDeviceToDevice, c->stream);
      // slot -1 of the local level-q cross array: S_{b_{r-1}, b_r} = boundary X_q slot r-1
      if (e == cudaSuccess) {
        if (c->small)   // tiled layouts: column r of the boundary's level-0 cross array -> local column 0
          e = cudaMemcpy2DAsync(c->Xq_local, 32 * 8, c->Xb[0] + (int64_t)(r >> 5) * 32 * nn + (r & 31), 32 * 8,
                                8, nn, cudaMemcpyDeviceToDevice, c->stream);
        else
          e = cudaMemcpyAsync(c->Xq_local, c->Xb[0] + (int64_t)r * nn, nn * 8, cudaMemcpyDeviceToDevice,
                              c->stream);
      }
    }
  }
  return cuda_fail(e);
}

}  // namespace

extern "C" {

int ks_dist_unique_id(unsigned char id[128]) {
  if (!id) return KS_ERR_ARG;
  if (!g_nccl.load()) return KS_ERR_NCCL;
  NcclUid u;
  if (g_nccl.uid(&u) != 0) return KS_ERR_NCCL;
  memcpy(id, u.internal, 128);
  return KS_OK;
}

int ks_dist_create(ks_dist **out, int rank, int nranks, const unsigned char *id, int64_t first_global_step,
                   int64_t nsteps_global) {
  if (!out) return KS_ERR_ARG;
  *out = nullptr;
  if (nranks < 1 || rank < 0 || rank >= nranks || nsteps_global < 1 || first_global_step < 0 ||
      first_global_step >= nsteps_global)
    return KS_ERR_ARG;
  ks_dist *d = new (std::nothrow) ks_dist;
  if (!d) return KS_ERR_ARG;
  d->rank = rank; d->nranks = nranks; d->first = first_global_step; d->nglobal = nsteps_global;
  if (id) {   // (a 1-rank communicator is legal: nothing to exchange, the library calls still run)
    if (!g_nccl.load()) { delete d; return KS_ERR_NCCL; }
    NcclUid u;
    memcpy(u.internal, id, 128);
    if (g_nccl.init(&d->comm, nranks, u, rank) != 0) { delete d; return KS_ERR_NCCL; }
  }
  *out = d;
  return KS_OK;
}

int ks_dist_info(const ks_dist *d, int *rank, int *nranks, int *nccl_nranks) {
  if (!d) return KS_ERR_ARG;
  if (rank) *rank = d->rank;
  if (nranks) *nranks = d->nranks;
  if (nccl_nranks) {
    *nccl_nranks = 0;
    if (d->comm && g_nccl.count(d->comm, nccl_nranks) != 0) return KS_ERR_NCCL;
  }
  return KS_OK;
}

void ks_dist_destroy(ks_dist *d) {
  if (!d) return;
  if (d->comm) g_nccl.destroy(d->comm);
  delete d;
}

size_t ks_workspace_bytes(const ks_problem *p, const ks_dist *d) {
  if (validate(p, d) != KS_OK) return 0;
  ks_ctx c;
  c.p = *p;
  c.N = p->nsteps; c.n = p->n; c.mx = p->m_max; c.rc = level0_rows(p);
  c.host_inputs = (p->flags & KS_HOST_INPUTS) != 0;
  c.small = use_small(p);
  c.big = use_big(p);
  c.seg = segment_steps(p, d);
  if (d && d->nranks > 1) {
    c.sharded = true; c.rank = d->rank; c.nranks = d->nranks;
    int q = 0;
    while ((1ll << q) < p->nsteps) ++q;
    c.q = q;
  }
  return carve(&c, nullptr) + kAlign;
}

int ks_create(ks_ctx **out, const ks_problem *p, void *workspace, size_t ws_bytes, void *stream,
              const ks_dist *d, double *states_out, double *cov_out) {
  if (!out) return KS_ERR_ARG;
  *out = nullptr;
  int v = validate(p, d);
  if (v) return v;
  if (!workspace || ((uintptr_t)workspace % kAlign) != 0) return KS_ERR_WORKSPACE;
  size_t need = ks_workspace_bytes(p, d);
  if (ws_bytes + kAlign < need) return KS_ERR_WORKSPACE;
  ks_ctx *c = new (std::nothrow) ks_ctx;
  if (!c) return KS_ERR_ARG;
  c->p = *p;
  c->N = p->nsteps; c->n = p->n; c->mx = p->m_max; c->rc = level0_rows(p);
  c->general = p->Hev || p->l || p->nstate;
  c->stream = (cudaStream_t)stream;
  c->host_inputs = (p->flags & KS_HOST_INPUTS) != 0;
  c->chol = (p->flags & KS_COV_IS_CHOL) != 0;
  c->seg = segment_steps(p, d);
  c->small = use_small(p);
  c->big = use_big(p);
  if (d && d->nranks > 1) {
    c->sharded = true; c->rank = d->rank; c->nranks = d->nranks; c->comm = d->comm;
    int q = 0;
    while ((1ll << q) < p->nsteps) ++q;
    c->q = q;
  }
  c->xout = states_out;
  c->Sout = cov_out;
  if ((p->flags & KS_OUTPUTS_BOUND) && !states_out) { delete c; return KS_ERR_ARG; }
  carve(c, (char *)workspace);
  if (c->host_inputs) {
    c->m = c->st_m; c->F = c->st_F; c->K = c->st_K; c->H = c->st_H; c->L = c->st_L;
    c->o = c->st_o; c->c = c->st_c; c->Hev = c->st_Hev; c->l = c->st_l; c->ns = c->st_ns;
  } else {
    c->m = p->m; c->F = p->F; c->K = p->K; c->H = p->H; c->L = p->L; c->o = p->o; c->c = p->c;
    c->Hev = p->Hev; c->l = p->l; c->ns = p->nstate;
  }
  if (c->big) {
    ks::big::Plan &b = c->bp;
    b.m = c->m; b.F = c->F; b.H = c->H; b.c = c->c; b.o = c->o; b.K = c->K; b.L = c->L;
    b.sF = p->sF; b.sH = p->sH; b.sc = p->sc; b.so = p->so; b.sK = p->sK; b.sL = p->sL;
    b.status = c->status;
    b.x = c->xout; b.S = c->Sout;
    // the second stream of the factor (stage 3 beside stage 2); its work is
    // ordered with the context's stream by events, so it is captured into
    // the same CUDA graph
    if (cudaStreamCreateWithFlags(&b.s2, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&b.ev[0], cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&b.ev[1], cudaEventDisableTiming) != cudaSuccess) {
      cudaGetLastError();
      b.s2 = nullptr;
    }
    // the QRs' lookahead side streams (one per QR stream), unless KS_NO_LOOKAHEAD
    if (!std::getenv("KS_NO_LOOKAHEAD"))
      for (ks::big::Work *wk : {&b.w, &b.w2})
        if (cudaStreamCreateWithFlags(&wk->side, cudaStreamNonBlocking) != cudaSuccess ||
            cudaEventCreateWithFlags(&wk->evf, cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&wk->evj, cudaEventDisableTiming) != cudaSuccess) {
          cudaGetLastError();
          wk->side = nullptr;
        }
  }
  *out = c;
  return KS_OK;
}

int ks_whiten(ks_ctx *c) {
  NvtxRange nvtx_("ks_whiten");
  if (!c) return KS_ERR_ARG;
  cudaError_t e = cudaMemsetAsync(c->status, 0xff, 16, c->stream);
  if (e != cudaSuccess) return cuda_fail(e);
  if (c->host_inputs) {
    const ks_problem &p = c->p;
    struct { void *d; const void *h; size_t bytes; } cp[] = {
        {c->st_m, p.m, p.m ? (size_t)c->N * 4 : 0}, {c->st_F, p.F, c->nF * 8}, {c->st_K, p.K, c->nK * 8},
        {c->st_H, p.H, c->nH * 8}, {c->st_L, p.L, c->nL * 8}, {c->st_o, p.o, c->no * 8},
        {c->st_c, p.c, c->nc * 8}, {c->st_Hev, p.Hev, c->nHev * 8},
        {c->st_l, p.l, p.l ? (size_t)c->N * 4 : 0}, {c->st_ns, p.nstate, p.nstate ? (size_t)c->N * 4 : 0}};
    for (auto &x : cp)
      if (x.bytes) {
        e = cudaMemcpyAsync(x.d, x.h, x.bytes, cudaMemcpyHostToDevice, c->stream);
        if (e != cudaSuccess) return cuda_fail(e);
      }
  }
  if (c->big) {
    const int64_t l0 = ks::big::g_launches.load();
    e = ks::big::whiten(c->bp, c->stream);
    c->launches += ks::big::g_launches.load() - l0;
    if (e != cudaSuccess) return cuda_fail(e);
    c->stage = 1;
    c->solved = c->covd = false;
    return KS_OK;
  }
  if (c->small) {
    SmallWhitenArgs a;
    a.N = c->N; a.n = c->n; a.m_max = c->mx; a.m = c->m;
    a.F = c->F; a.H = c->H; a.c = c->c; a.o = c->o; a.K = c->K; a.L = c->L;
    a.sF = c->p.sF; a.sH = c->p.sH; a.sc = c->p.sc; a.so = c->p.so; a.sK = c->p.sK; a.sL = c->p.sL;
    a.first_global = c->sharded ? (int64_t)c->rank * c->N : 0;
    a.cntE = c->cntE; a.cntC = c->cntC;
    a.constC = c->constC;
    const SmallIn v = small_level0(c);
    a.C = v.C; a.y = v.y; a.El = v.El; a.Er = v.Er; a.e = v.e; a.nC = v.nC; a.nEr = v.nEr; a.nEl = v.nEl;
    a.cE = c->cntE == 1;
    a.cC = c->cntC == 1;
    a.Mchol = c->Mchol; a.status = c->status;
    a.Minv = small_yfuse(c) ? c->Minv : nullptr;
    a.chol = c->chol;
    a.seg = c->seg;
    a.Mall = c->Mall;
    a.Hev = c->Hev; a.sHev = c->p.sHev; a.l = c->l; a.ns = c->ns; a.RC = c->rc;
    int nl = 0;
    {
      Launch l(c, 0, 0, 1);
      e = launch_small_whiten(a, c->stream, &nl);
    }
    if (e != cudaSuccess) return cuda_fail(e);
    c->stage = 1;
    c->solved = c->covd = false;
    return KS_OK;
  }
  WhitenArgs a;
  a.N = c->N; a.n = c->n; a.m_max = c->mx; a.m = c->m;
  a.F = c->F; a.H = c->H; a.c = c->c; a.o = c->o; a.K = c->K; a.L = c->L;
  a.sF = c->p.sF; a.sH = c->p.sH; a.sc = c->p.sc; a.so = c->p.so; a.sK = c->p.sK; a.sL = c->p.sL;
  a.first_global = c->sharded ? (int64_t)c->rank * c->N : 0;
  a.C = c->C0; a.y = c->y0; a.El = c->El0; a.Er = c->Er0; a.e = c->e0;
  a.cntE = c->cntE; a.cntC = c->cntC; a.Mchol = c->Mchol; a.status = c->status;
  a.chol = c->chol;
  a.seg = c->seg;
  a.Mall = c->Mall;
  a.Hev = c->Hev; a.sHev = c->p.sHev; a.l = c->l; a.ns = c->ns; a.RC = c->rc;
  a.constC = c->constC;
  {
    Launch l(c, 0, 0, 1 + (c->rc > 0) + (c->mx > 0 && c->constC));
    e = launch_whiten(a, c->stream);
  }
  if (e != cudaSuccess) return cuda_fail(e);
  c->stage = 1;
  c->solved = c->covd = false;
  return KS_OK;
}

int ks_factor(ks_ctx *c) {
  NvtxRange nvtx_("ks_factor");
  if (!c) return KS_ERR_ARG;
  if (c->stage < 1) return KS_ERR_ORDER;
  if (c->big) {
    const int64_t l0 = ks::big::g_launches.load();
    Launch l(c, 1, 0, 0);
    cudaError_t e = ks::big::factor(c->bp, c->stream);
    c->launches += ks::big::g_launches.load() - l0;
    if (e != cudaSuccess) return cuda_fail(e);
    c->stage = 3;
    return KS_OK;
  }
  int r = run_factor_levels(c, false);
  if (r) return r;
  if (!c->sharded) {
    c->stage = 3;
    return KS_OK;
  }
  c->stage = 2;
  if (!c->comm) return KS_OK;  // caller-driven exchange: ks_boundary_buffers + ks_factor_boundary
  const size_t E = (size_t)entry_doubles(c->n);
  int rc = g_nccl.allgather(c->send, c->recv, E, /*ncclFloat64*/ 8, c->comm, c->stream);
  if (rc != 0) return KS_ERR_NCCL;
  return ks_factor_boundary(c);
}

int ks_boundary_buffers(ks_ctx *c, void **send, void **recv, size_t *bytes) {
  if (!c || !c->sharded) return KS_ERR_ARG;
  if (send) *send = c->send;
  if (recv) *recv = c->recv;
  if (bytes) *bytes = (size_t)entry_doubles(c->n) * 8;
  return KS_OK;
}

int ks_factor_boundary(ks_ctx *c) {
  NvtxRange nvtx_("ks_factor_boundary");
  if (!c || !c->sharded) return KS_ERR_ARG;
  if (c->stage != 2) return KS_ERR_ORDER;
  int r = run_factor_levels(c, true);
  if (r) return r;
  c->stage = 3;
  return KS_OK;
}

// the large-n path's backward phases
static int big_backward(ks_ctx *c, bool st, bool cov) {
  const int64_t l0 = ks::big::g_launches.load();
  cudaError_t e;
  {
    Launch l(c, (cov && st) ? 5 : (cov ? 3 : 2), 0, 0);
    e = ks::big::backward(c->bp, st, cov, c->stream);
  }
  c->launches += ks::big::g_launches.load() - l0;
  if (e != cudaSuccess) return cuda_fail(e);
  if (st) c->solved = true;
  if (cov) c->covd = true;
  return KS_OK;
}

int ks_solve(ks_ctx *c) {
  NvtxRange nvtx_("ks_solve");
  if (!c) return KS_ERR_ARG;
  if (c->stage < 3) return KS_ERR_ORDER;
  if (c->big) return big_backward(c, true, false);
  int r;
  if (c->sharded) {
    if ((r = run_backward_levels(c, true, 1, 0))) return r;
    if ((r = scatter_boundary(c, true, false))) return r;
  }
  if ((r = run_backward_levels(c, false, 1, 0))) return r;
  c->solved = true;
  return KS_OK;
}

int ks_selinv(ks_ctx *c) {
  NvtxRange nvtx_("ks_selinv");
  if (!c || !c->Sout) return KS_ERR_ARG;
  if (c->stage < 3) return KS_ERR_ORDER;
  if (c->big) return big_backward(c, false, true);
  int r;
  if (c->sharded) {
    if ((r = run_backward_levels(c, true, 0, 1))) return r;
    if ((r = scatter_boundary(c, false, true))) return r;
  }
  if ((r = run_backward_levels(c, false, 0, 1))) return r;
  c->covd = true;
  return KS_OK;
}

int ks_solve_selinv(ks_ctx *c) {
  NvtxRange nvtx_("ks_solve_selinv");
  if (!c || !c->Sout) return KS_ERR_ARG;
  if (c->stage < 3) return KS_ERR_ORDER;
  if (c->big) return big_backward(c, true, true);
  int r;
  if (c->sharded) {
    if ((r = run_backward_levels(c, true, 1, 1))) return r;
    if ((r = scatter_boundary(c, true, true))) return r;
  }
  if ((r = run_backward_levels(c, false, 1, 1))) return r;
  c->solved = c->covd = true;
  return KS_OK;
}

int ks_update_obs(ks_ctx *c, const double *o) {
  NvtxRange nvtx_("ks_update_obs");
  if (!c || (!o && c->mx > 0)) return KS_ERR_ARG;
  if (c->stage < 1) return KS_ERR_ORDER;
  const bool constC = c->constC;
  if (c->big) return KS_ERR_ARG;                 // not on the large-n path
  if (!constC && !c->Mall) return KS_ERR_ARG;   // needs KS_KEEP_WHITENING
  if (c->mx > 0) {
    cudaError_t e = cudaSuccess;
    if (c->host_inputs) {   // the new observations into the staging buffer (H2D)
      e = cudaMemcpyAsync(c->st_o, o, c->no * 8, cudaMemcpyHostToDevice, c->stream);
      if (e != cudaSuccess) return cuda_fail(e);
    } else {
      c->o = o;
      c->p.o = o;
    }
    if (!(c->small && small_yfuse(c))) {   // (fused y: the factor whitens o itself)
      Launch l(c, 0, 0, 1);
      e = launch_update_y(constC ? c->Mchol : c->Mall, constC ? 0 : (int64_t)c->mx * c->mx, c->o, c->p.so, c->m,
                          c->mx, c->rc, c->N, c->y0, c->small ? 1 : 0, c->stream);
      if (e != cudaSuccess) return cuda_fail(e);
    }
  }
  c->stage = 1;
  c->solved = false;   // covariances do not depend on o: c->covd stays
  return KS_OK;
}

static int get_impl(ks_ctx *c, double *states, double *cov, bool sync_host);

int ks_get(ks_ctx *c, double *states, double *cov) { return get_impl(c, states, cov, true); }

namespace {
// S (N x n x n, row-major blocks) -> the upper triangles by rows (ks_get_packed)
__global__ void pack_cov_kernel(const double *__restrict__ S, int64_t N, int n, double *__restrict__ out) {
  const int P = n * (n + 1) / 2;
  const int64_t total = N * P;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = idx / P;
    int rem = (int)(idx - i * P), r = 0;
    while (rem >= n - r) {
      rem -= n - r;
      ++r;
    }
    out[idx] = __ldg(S + i * n * n + (int64_t)r * n + r + rem);
  }
}
}  // namespace

int ks_get_packed(ks_ctx *c, double *states, double *cov_packed, int sync) {
  if (!c) return KS_ERR_ARG;
  if ((states && !c->solved) || (cov_packed && !c->covd)) return KS_ERR_ORDER;
  double *dst = cov_packed;
  bool host = false;
  if (cov_packed) {
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, cov_packed) != cudaSuccess) {
      cudaGetLastError();
      return KS_ERR_ARG;
    }
    if (at.type == cudaMemoryTypeHost) {   // page-locked: the kernel writes through its device alias
      if (!at.devicePointer) return KS_ERR_ARG;
      dst = (double *)at.devicePointer;
      host = true;
    } else if (at.type != cudaMemoryTypeDevice && at.type != cudaMemoryTypeManaged) {
      return KS_ERR_ARG;   // pageable host memory
    }
  }
  int r = get_impl(c, states, nullptr, false);
  if (r != KS_OK) return r;
  if (cov_packed && c->N > 0) {
    int dev = 0, sms = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t total = c->N * (int64_t)(c->n * (c->n + 1) / 2);
    const int64_t blocks = std::min<int64_t>((total + 255) / 256, (int64_t)sms * 8);
    pack_cov_kernel<<<(unsigned)blocks, 256, 0, c->stream>>>(c->Sout, c->N, c->n, dst);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e);
  }
  if (sync) {
    bool hs = host;
    if (states) {
      cudaPointerAttributes at;
      if (cudaPointerGetAttributes(&at, states) != cudaSuccess) { cudaGetLastError(); hs = true; }
      else if (at.type != cudaMemoryTypeDevice && at.type != cudaMemoryTypeManaged) hs = true;
    }
    if (hs) return cuda_fail(cudaStreamSynchronize(c->stream));
  }
  return KS_OK;
}

int ks_get_async(ks_ctx *c, double *states, double *cov) { return get_impl(c, states, cov, false); }

static int get_impl(ks_ctx *c, double *states, double *cov, bool sync_host) {
  if (!c) return KS_ERR_ARG;
  if ((states && !c->solved) || (cov && !c->covd)) return KS_ERR_ORDER;
  bool host = false;
  cudaError_t e = cudaSuccess;
  auto copy = [&](double *dst, const double *src, size_t bytes) {
    if (!dst || dst == src || e != cudaSuccess) return;
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, dst) != cudaSuccess) { cudaGetLastError(); at.type = cudaMemoryTypeUnregistered; }
    if (at.type != cudaMemoryTypeDevice && at.type != cudaMemoryTypeManaged) host = true;
    e = cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, c->stream);
  };
  copy(states, c->xout, (size_t)c->N * c->n * 8);
  copy(cov, c->Sout, (size_t)c->N * c->n * c->n * 8);
  if (e == cudaSuccess && host && sync_host) e = cudaStreamSynchronize(c->stream);
  return cuda_fail(e);
}

int ks_sync_status(ks_ctx *c, int64_t *bad_step, int *bad_kind) {
  if (!c) return KS_ERR_ARG;
  if (bad_step) *bad_step = -1;
  if (bad_kind) *bad_kind = 0;
  cudaError_t e = cudaStreamSynchronize(c->stream);
  if (e != cudaSuccess) return cuda_fail(e);
  unsigned long long st = 0;
  e = cudaMemcpy(&st, c->status, 8, cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return cuda_fail(e);
  if (st == kStatusOk) return KS_OK;
  const int kind = (int)(st & 0xff);
  if (bad_step) *bad_step = status_step(st);
  if (kind == kBadRank) return KS_ERR_RANK;
  if (kind == kBadScale) {   // small path: whitened data outside its exponent range
    if (bad_kind) *bad_kind = 3;
    return KS_ERR_ARG;
  }
  if (bad_kind) *bad_kind = kind;
  return KS_ERR_NOT_SPD;
}

int ks_set_timing(ks_ctx *c, int on) {
  if (!c) return KS_ERR_ARG;
  cudaError_t e = cudaStreamSynchronize(c->stream);
  if (e != cudaSuccess) return cuda_fail(e);
  c->timing = on != 0;
  c->ev_used = 0;
  c->ev_family.clear();
  c->ev_level.clear();
  c->rec_family.clear();
  c->rec_level.clear();
  c->rec_ms.clear();
  for (int f = 0; f < KS_NFAMILIES; ++f) { c->t_ms[f] = 0; c->t_cnt[f] = 0; }
  return KS_OK;
}

namespace {
int drain_events(ks_ctx *c) {
  cudaError_t e = cudaStreamSynchronize(c->stream);
  if (e != cudaSuccess) return cuda_fail(e);
  for (size_t i = 0; i < c->ev_family.size(); ++i) {
    float t = 0.f;
    cudaEventElapsedTime(&t, c->ev_pool[2 * i], c->ev_pool[2 * i + 1]);
    c->t_ms[c->ev_family[i]] += t;
    c->t_cnt[c->ev_family[i]] += 1;
    c->rec_family.push_back(c->ev_family[i]);
    c->rec_level.push_back(c->ev_level[i]);
    c->rec_ms.push_back(t);
  }
  c->ev_used = 0;
  c->ev_family.clear();
  c->ev_level.clear();
  return KS_OK;
}
}  // namespace

int ks_get_timing(ks_ctx *c, double ms[KS_NFAMILIES], int64_t launches[KS_NFAMILIES]) {
  if (!c) return KS_ERR_ARG;
  int r = drain_events(c);
  if (r) return r;
  for (int f = 0; f < KS_NFAMILIES; ++f) {
    if (ms) ms[f] = c->t_ms[f];
    if (launches) launches[f] = c->t_cnt[f];
  }
  return KS_OK;
}

int64_t ks_get_launch_times(ks_ctx *c, int64_t cap, int32_t *family, int32_t *level, float *ms) {
  if (!c) return -KS_ERR_ARG;
  int r = drain_events(c);
  if (r) return -r;
  const int64_t cnt = (int64_t)c->rec_ms.size();
  for (int64_t i = 0; i < cnt && i < cap; ++i) {
    if (family) family[i] = c->rec_family[i];
    if (level) level[i] = c->rec_level[i];
    if (ms) ms[i] = c->rec_ms[i];
  }
  return cnt;
}

int ks_info(ks_ctx *c, int64_t *levels, int64_t *launches) {
  if (!c) return KS_ERR_ARG;
  if (levels) *levels = (int64_t)c->K_.size() + (int64_t)c->Kb.size();
  if (launches) *launches = c->launches;
  return KS_OK;
}

int ks_level_of_steps(int64_t N, int32_t *level) {
  if (N < 1) return -KS_ERR_ARG;
  const std::vector<int64_t> Ks = level_sizes(N, -1);
  for (size_t L = 0; L < Ks.size(); ++L)
    for (int64_t t = 0; t < Ks[L]; t += 2)
      if (level) level[((t + 1) << L) - 1] = (int32_t)L;
  return (int)Ks.size();
}

const char *ks_strerror(int code) {
  switch (code) {
    case KS_OK: return "ok";
    case KS_ERR_ARG: return "bad argument";
    case KS_ERR_ORDER: return "call out of order";
    case KS_ERR_CUDA: return "CUDA error";
    case KS_ERR_NCCL: return "NCCL unavailable or failed";
    case KS_ERR_NOT_SPD: return "noise covariance not SPD";
    case KS_ERR_RANK: return "least-squares matrix rank deficient";
    case KS_ERR_WORKSPACE: return "workspace too small or misaligned";
    default: return "unknown";
  }
}

void ks_destroy(ks_ctx *c) {
  if (!c) return;
  if (c->big) {
    if (c->bp.s2) cudaStreamDestroy(c->bp.s2);
    for (cudaEvent_t e : c->bp.ev)
      if (e) cudaEventDestroy(e);
    for (ks::big::Work *wk : {&c->bp.w, &c->bp.w2}) {
      if (wk->side) cudaStreamDestroy(wk->side);
      if (wk->evf) cudaEventDestroy(wk->evf);
      if (wk->evj) cudaEventDestroy(wk->evj);
    }
  }
  for (auto e : c->ev_pool) cudaEventDestroy(e);
  delete c;
}

}  // extern "C"
