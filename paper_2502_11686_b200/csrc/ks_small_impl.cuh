// Small-n path implementation (templates); instantiated per n by ks_small_n<n>.cu
// so that the eight state dimensions compile in parallel.
#pragma once
// Small-n path (n <= 8, m_max <= 8) of the Odd-Even Kalman smoother.
//
// One THREAD per (even, odd) column pair / per eliminated column, every block
// held in registers (the state dimension N is a template parameter, so all
// loops unroll and all block indices are compile-time), and every block QR
// done by Givens row streaming into a packed upper-triangular R: a stacked
// QR [R; rows] is computed by rotating one row at a time into R.  Givens and
// Householder produce the same R up to row signs (both are Q R of the same
// stack), and the row-streaming form needs only one streamed row
// in registers at a time instead of the whole (2n+m) x (3n+1) stack, which is
// what lets a whole pair fit in one thread's registers.  Level arrays are
// element-major (SoA), so the 32 threads of a warp load element e of 32
// consecutive columns with one coalesced 256-byte access.
//
// P:n = line n of the paper text.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <type_traits>

#include "ks_internal.cuh"

#ifndef KS_PF_ROWS
#define KS_PF_ROWS 2   // L1 prefetch distance of the streamed rows
#endif
#ifndef KS_BWD_TMA
#define KS_BWD_TMA 1   // regular backward levels of even n: TMA tensor copies
#endif
#ifndef KS_TMAP_PROMO
#define KS_TMAP_PROMO CU_TENSOR_MAP_L2_PROMOTION_L2_64B   // L2 promotion of the backward TMA rows: 64 B (A/B: 256 B 0.605 ms, none 0.586, 64 B 0.569 at c5 backward L0)
#endif
#ifndef KS_F6_L0C_BLOCKS
#define KS_F6_L0C_BLOCKS 6
#endif
#ifndef KS_F6_BLOCKS
#define KS_F6_BLOCKS 4
#endif

namespace ks {
namespace smalld {

template <int N>
struct Tri {
  static constexpr int size = N * (N + 1) / 2;
  static constexpr __host__ __device__ int at(int i, int j) { return i * N - (i * (i - 1)) / 2 + (j - i); }
};

// Column base of a tiled (ES = 32), pair-interleaved tiled (ES = 64) or
// AoS / constant (ES = 1) view; element e of the column is then at
// base[EST * e] (EST = 32 for both tiled layouts), a compile-time immediate.
//   ES = 32: p[(t >> 5) ts + 32 e + (t & 31)]
//   ES = 64: p[(t >> 6) ts + (t & 1) ts/2 + 32 e + ((t >> 1) & 31)]
// The pair-interleaved layout keeps the even and the odd columns of each 64
// in separate 32-column halves, so that a warp of pair threads reading
// column 2p (or 2p+1) of 32 consecutive pairs touches 256 contiguous bytes.
template <int ES>
__device__ __forceinline__ double *cb(const TView &v, int64_t t) {
  if (ES == 64) return v.p + (t >> 6) * v.ts + (t & 1) * (v.ts >> 1) + ((t >> 1) & 31);
  return ES == 32 ? v.p + (t >> 5) * v.ts + (t & 31) : v.p + t * v.ts;
}
template <int ES>
__host__ __device__ constexpr int est() { return ES == 64 ? 32 : ES; }
template <int ES>
__device__ __forceinline__ double ldv(const TView &v, int64_t t, int e) {
  return __ldg(cb<ES>(v, t) + est<ES>() * e);
}
template <int ES>
__device__ __forceinline__ void stv(const TView &v, int64_t t, int e, double x) {
  cb<ES>(v, t)[est<ES>() * e] = x;
}
// L1 prefetch of element e of column t (no registers): the row loops fetch
// the next streamed rows while rotating the current one.
template <int ES>
__device__ __forceinline__ void pfv(const TView &v, int64_t t, int e) {
  asm volatile("prefetch.global.L1 [%0];" ::"l"(cb<ES>(v, t) + est<ES>() * e));
}

// L1 prefetch of the 128-byte line holding p
__device__ __forceinline__ void pf_line(const double *p) { asm volatile("prefetch.global.L1 [%0];" ::"l"(p)); }

__device__ __forceinline__ void report(unsigned long long *st, int64_t step, int kind) {
  if (st) atomicMin(st, status_word(step, kind));
}

// 1/sqrt(h) for h > 0: the MUFU approximation refined by two Newton steps
// (each doubles the correct bits: ~2^-22 -> ~2^-44 -> full double).  No
// special-case branches.
__device__ __forceinline__ double rsqrt_nr(double h) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(h));
  double hy = h * y;
  y = fma(0.5 * y, fma(-hy, y, 1.0), y);
  hy = h * y;
  y = fma(0.5 * y, fma(-hy, y, 1.0), y);
  return y;
}
// sqrt(h) for h >= 0 (0 -> 0), branch-free.
__device__ __forceinline__ double sqrt_nr(double h) {
  const bool z = !(h > 0.0);
  const double r = h * rsqrt_nr(z ? 1.0 : h);
  return z ? 0.0 : r;
}
// 1/x for x != 0: the MUFU approximation (relative error <= 2^-19.9,
// measured on B200: tools/micro/rcp_bench.cu) refined by one third-order
// Newton step y' = y + y (e + e^2), e = 1 - x y: error ~e^3 < 2^-59.
__device__ __forceinline__ double rcp_nr(double x) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double e = fma(-x, y, 1.0);
  return fma(y, fma(e, e, e), y);
}

// Square-root-free Givens rotations (Gentleman, 1973), in inverse-weight
// form.  Every row of the triangular factor is kept as
// R_k = sqrt(d_k) [1, u_{k,k+1}, ..., | trailing columns] and stored through
// rho_k = 1/d_k; every streamed row as sqrt(delta) [y_k, y_{k+1}, ...],
// stored through w = 1/delta.  Zeroing y_k against row k is the plane
// rotation with c = sqrt(d/d'), s = sqrt(delta) y_k / sqrt(d') (the same
// orthogonal Q as the classical Givens / Householder QR of P:424-436, up to
// row signs: R_kk = +sqrt(d_k)).  With d' = d + delta y_k^2:
//     w'   = w + y_k^2 rho                 (= 1/delta', delta' = delta d/d')
//     rho' = rho w / w',   sbar = y_k rho / w'   (= delta y_k / d')
//     y_j' = y_j - y_k u_j,  u_j' = u_j + sbar y_j'      (every column j > k)
// TWO fma per element and pair instead of four, one reciprocal per rotation,
// and -- the point of the inverse-weight form -- the serial dependence from
// one pivot to the next is a single fma (w') instead of a reciprocal (square
// root) chain: the reciprocals of consecutive pivots overlap.
//
// Empty rows.  A row of R that has received no data yet (level 0: R starts
// empty; m_i < n leaves rows empty after the observation rows) has
// rho = kEmptyRow, a huge FINITE value (d = 2^-600 ~ 2.4e-181, an initial row
// weight far below any data), so absorbing a streamed row into it is the same
// select-free rotation: with y_k != 0, sbar = (1/y_k)(1 - eps),
// rho' = (w/y_k^2)(1 - eps), w' ~ 2^600 y_k^2 (the streamed row is consumed:
// later rotations of it are the identity to eps), eps = w / (y_k^2 rho)
// < 1e-100 for every |y_k| >= 1e-40.  y_k = 0 (zero padding rows) leaves the
// row unchanged up to an ulp of rho.  Rows still empty at the end (rank
// deficiency) keep rho ~ 2^600 and fail the rank test.  One branch-free form
// for every rotation: no guards, one code path (half the code of a guarded
// version, and the compiler interleaves consecutive pivots).
constexpr double kEmptyRow = 0x1p600;
__device__ __forceinline__ void gmake(double &rho, double yk, double &w, double &sb) {
  const double yr = yk * rho;
  const double wn = fma(yk, yr, w);
  const double q = rcp_nr(wn);
  sb = yr * q;
  rho = rho * (w * q);
  w = wn;
}
// sqrt(delta) = 1/sqrt(w) of a streamed row.
__device__ __forceinline__ double wscale(double w) { return rsqrt_nr(w); }
// Apply to one column: u (row of R) and y (streamed row), yk the pivot value
// of the streamed row before the rotation.
__device__ __forceinline__ void gapp(double &u, double &y, double yk, double sb) {
  y = fma(-yk, u, y);
  u = fma(sb, y, u);
}

// A streamed row absorbed by an empty row of R (w ~ 2^600 y_k^2, see above)
// is consumed: its later rotations are the identity to eps, and as a stage-1
// leftover it carries no row of D~ (level 0 with m_i < n: the first n - m_i
// evolution rows fill the empty rows of R), so stage 3 skips it.  (Stopping
// the rotations of a row at its absorption was measured slower: the per-pivot
// exit branch serialises the overlapped reciprocals of consecutive pivots.)
constexpr double kConsumed = 0x1p500;
// Rotate one streamed row into R (row streaming): pivot part
// row[0..N), weight w; trail(k, y_k, sbar) applies rotation k to the row's
// trailing columns.
template <int N, class Trail>
__device__ __forceinline__ void rot_row(double (&R)[Tri<N>::size], double (&row)[N], double &w, Trail &&trail) {
#pragma unroll
  for (int k = 0; k < N; ++k) {
    double sb;
    const double yk = row[k];
    gmake(R[Tri<N>::at(k, k)], yk, w, sb);
#pragma unroll
    for (int j = k + 1; j < N; ++j) gapp(R[Tri<N>::at(k, j)], row[j], yk, sb);
    trail(k, yk, sb);
  }
}

// ---------------------------------------------------------------- factor ---

// Eliminate column t of the level in one thread.
//   stage 1: rotate the rows of [El_{t+1} | Er_{t+1} | e_{t+1}] into
//            R = C_t (level 0: the rows of C_t into R = 0 first), giving R~_t,
//            X_t, z~_t; each leftover row [0 | d | y~] (a row of D~_{t+1})
//   stage 3: is rotated at once into R3 = C_{t+1}, giving the survivor's
//            C'_{t+1} (plus the leftover Z rows of an odd level's last column)
//   stage 2: rotate the rows of [Er_t | El_t | 0 | e_t] into [R~_t | 0 | X_t | z~_t]
//            giving R_tt, R_{t,t-1}, R_{t,t+1}, z_t; the leftover rows are the
//            survivor's new coupling row [Z_t | X~_t | z^_t].  No left
//            neighbour: "nothing to do".
//   post:    T_l = R^{-1} R_{t,t-1}, T_r = R^{-1} R_{t,t+1}, w = R^{-1} z_t,
//            P = R^{-1} R^{-T} (packed) -> R record.
// All QRs are square-root-free Givens row streaming (gmake / gapp above), so
// R = D^{1/2} U with U unit upper triangular and the trailing blocks carry the
// same D^{1/2}: T = U^{-1} X needs no division and P = U^{-1} D^{-1} U^{-T}.
// Level >= 1 C-like blocks are stored in that form (1/d_k on the diagonal, U
// strictly above, y = D^{-1/2} z); coupling rows are stored as true rows
// (weight folded in: sqrt(delta) x row), so no weight accumulates over levels.
// Entry element offsets (entry_doubles layout).
template <int N>
struct Ent {
  static constexpr int C = 0, y = N * N, El = N * N + N, Er = 2 * N * N + N, e = 3 * N * N + N,
                       nrm = 3 * N * N + 2 * N;
};
// R record element offsets.
template <int N>
struct Rr {
  static constexpr int Tl = 0, Tr = N * N, w = 2 * N * N, P = 2 * N * N + N;
};

// Shared memory of the factor kernel: per-thread parking (leftover rows with
// their weights N(N+2) + R~ packed N(N+1)/2, element-major), then the staged
// constant level-0 blocks (El, Er, e, C with RC <= kSmallMaxM rows).
template <int N>
constexpr int kParkDoubles = N * (N + 2) + N * (N + 1) / 2;
// the split form (three threads per pair) also parks stage 1's z~_t for pass A's thread
template <int N>
constexpr int kParkSP = kParkDoubles<N> + N;
constexpr int kTailThreads = 192;   // split form: three threads (roles) per pair slot
template <int N>
struct CstOff {
  static constexpr int El = 0, Er = N * N, e = 2 * N * N, C = 2 * N * N + N,
                       Mi = 2 * N * N + N + kSmallMaxM * N,   // M^{-1} (constant observation model)
      size = 2 * N * N + N + kSmallMaxM * N + kSmallMaxM * kSmallMaxM;
};

// SPL (the fused tail and latency-bound levels): the pair's work is split over three
// threads of one slot -- role 0 stage 1 + pass B (+ T_r), role 1 stage 3,
// role 2 pass A + post -- which meet at two CTA barriers (after stage 1's
// parking, at the end); `active` false only joins the barriers.  Same
// operations in the same order per result as the one-thread form (bitwise).
template <int N, bool L0, bool CE, bool CC, bool OAOS, bool SIN = false, bool ZS = false, bool SPL = false>
__device__ __forceinline__ void small_eliminate(const SmallFactorArgs &a, int64_t t, bool hr, bool hl,
                                                int64_t pnext, bool zs_in, bool zs_out,
                                                volatile int *zsync = nullptr, int zval = 0, int role = 0,
                                                int slot = 0, bool active = true) {
  using TR = Tri<N>;
#ifndef KS_ROW_UNROLL
#define KS_ROW_UNROLL 1
#endif
  constexpr int UR = KS_ROW_UNROLL;   // row loops stay rolled: the unrolled body thrashes the I-cache
  using EN = Ent<N>;
  using RR = Rr<N>;
  const SmallIn &in = a.in;
  double *zs_ = a.zscratch;
  // level >= 1 entry element e of column c: read-only global (__ldg), or
  // shared memory (SIN: the fused tail kernel keeps its levels on chip)
  auto lde = [&](int64_t c, int e) {
    return SIN ? cb<64>(in.ent, c - a.ent_off)[32 * e] : ldv<64>(in.ent, c, e);
  };
  // field loads: level 0 per-field views (constant blocks: ES = 1, ts = 0),
  // level >= 1 one tiled entry record view
  constexpr int ESE = CE ? 1 : 64, ESC = CC ? 1 : 64, ESO = OAOS ? 1 : 64;
  // constant level-0 blocks (stride-0 model) are staged once per CTA in
  // shared memory by the kernel prologue and read there (broadcast)
  extern __shared__ double smem_park[];
  const double *cst = smem_park + (SPL ? (size_t)64 * kParkSP<N> : (size_t)blockDim.x * kParkDoubles<N>);
  // roles (SPL): r0 stage 1 + pass B, r1 stage 3, r2 pass A + post
  const bool r0 = !SPL || (active && role == 0), r1 = !SPL || (active && role == 1),
             r2 = !SPL || (active && role == 2);
  auto split_bar = [&](int id) {
    if (SPL) asm volatile("barrier.sync %0, 192;" ::"r"(id) : "memory");   // one call site each
  };
  auto ldC = [&](int e, int64_t c) {
    return L0 ? (CC ? cst[CstOff<N>::C + e] : ldv<64>(in.C, c, e)) : lde(c, EN::C + e);
  };
  // level-0 observations: y = M^{-1} o computed here for a
  // constant observation model (M^{-1} staged in shared memory), else the
  // whitened y of ks_whiten
  auto ldY = [&](int e, int64_t c) {
    if (!L0) return lde(c, EN::y + e);
    if (CC && in.yfuse) {
      // y_e = sum_k (M^{-1})_{ek} o_k over k < RC (M^{-1} is lower triangular:
      // the terms k > e add exact zeros), unrolled so that the loads of o
      // issue together instead of one dependent load per iteration
      const double *oc = in.o + c * in.so;
      double yv = 0.0;
#pragma unroll
      for (int k = 0; k < kSmallMaxM; ++k)
        if (k < in.RC) yv = fma(cst[CstOff<N>::Mi + e * kSmallMaxM + k], __ldg(oc + k), yv);
      return yv;
    }
    return ldv<64>(in.y, c, e);
  };
  auto ldEl = [&](int e, int64_t c) {
    return L0 ? (CE ? cst[CstOff<N>::El + e] : ldv<64>(in.El, c, e)) : lde(c, EN::El + e);
  };
  auto ldEr = [&](int e, int64_t c) {
    return L0 ? (CE ? cst[CstOff<N>::Er + e] : ldv<64>(in.Er, c, e)) : lde(c, EN::Er + e);
  };
  auto ldE = [&](int e, int64_t c) {
    return L0 ? (CE ? cst[CstOff<N>::e + e] : ldv<64>(in.e, c, e)) : lde(c, EN::e + e);
  };
  // survivor entry store; the fused tail's last level may write the sharded
  // rank's AoS boundary send entry (a.outAoS, a runtime choice there only)
  auto sto = [&](int e, double v) {
    if (SIN && a.outAoS) a.out.p[(pnext - a.out_off) * a.out.ts + e] = v;
    else stv<ESO>(a.out, pnext - a.out_off, e, v);
  };
  // prefetch row i of a block field (n elements per row) of column c
  auto pfEl = [&](int i, int64_t c) {
#pragma unroll
    for (int j = 0; j < N; ++j) {
      if (!L0 && !SIN) pfv<64>(in.ent, c, EN::El + i * N + j);
      else if (!CE) pfv<64>(in.El, c, i * N + j);
    }
  };
  auto pfEr = [&](int i, int64_t c) {
#pragma unroll
    for (int j = 0; j < N; ++j) {
      if (!L0 && !SIN) pfv<64>(in.ent, c, EN::Er + i * N + j);
      else if (!CE) pfv<64>(in.Er, c, i * N + j);
    }
  };
  const int64_t rcol = t >> 1;
  auto str = [&](int e, double v) { stv<32>(a.rec, rcol, e, v); };
  double R[TR::size];   // d_k on the diagonal, U strictly above
  double X[N][N];
  double z[N];

  // rank reference: |block column of UA|_F (reading R9)
  double ref2 = 1.0, ref2u = 0.0;
  if (SPL && !active) {
  } else if (!L0) {
    const double v = lde(t, EN::nrm);
    ref2 = v * v;
    if (hr) {
      const double u = lde(t + 1, EN::nrm);
      ref2u = u * u;
    }
  } else {
    ref2 = ldv<ESC>(in.nC, t, 0) + (hl ? ldv<ESE>(in.nEr, t, 0) : 0.0) +
           (hr ? ldv<ESE>(in.nEl, t + 1, 0) : 0.0);
    if (hr)
      ref2u = ldv<ESC>(in.nC, t + 1, 0) + ldv<ESE>(in.nEr, t + 1, 0) +
              (t + 2 < a.K ? ldv<ESE>(in.nEl, t + 2, 0) : 0.0);
  }

#pragma unroll
  for (int i = 0; i < N; ++i) {
    z[i] = 0.0;
#pragma unroll
    for (int j = 0; j < N; ++j) X[i][j] = 0.0;
  }
  // Per-thread shared-memory parking (element-major: element e of this
  // thread at sp[e * blockDim.x]): the stage-1 leftover rows with their
  // weights (N x (N+2)) and a copy of R~_t (packed), so that at most ~76
  // doubles are live in registers at any point (stage 1 -> stage 2 pass B ->
  // stage 3 -> pass A).
  double *sp = smem_park + (SPL ? slot : threadIdx.x);
  const int bs = SPL ? 64 : blockDim.x;
  auto park = [&](int e, double v) { sp[e * bs] = v; };
  auto unpark = [&](int e) { return sp[e * bs]; };
  constexpr int kLeft = 0, kRt = N * (N + 2);

  // stream one weighted row [row (pivot part, N) | rhs] into (Rm, zm)
  auto stream_row = [&](double(&Rm)[TR::size], double(&zm)[N], double(&row)[N], double &rhs, double wl) {
    rot_row<N>(Rm, row, wl, [&](int k, double yk, double sb) { gapp(zm[k], rhs, yk, sb); });
  };

  // ---- stage 1 base: R = C_t ----
  // Prefetch into L1 what the stage-1 base and stage 3 read first (their row
  // loops are rolled, so each row's loads would otherwise wait a full memory
  // round trip): the observations (and per-step C rows) of both columns at
  // level 0, C_t / y_t of the entry at level >= 1 (C_{t+1} / y_{t+1}: pass B).
  if (L0) {
    if (CC && in.yfuse) {
      pf_line(in.o + t * in.so);
      if (hr) pf_line(in.o + (t + 1) * in.so);
    }
#pragma unroll 1
    for (int r = 0; r < in.RC; ++r) {
      if (!(CC && in.yfuse)) {
        pfv<64>(in.y, t, r);
        if (hr) pfv<64>(in.y, t + 1, r);
      }
      if (!CC) {
#pragma unroll
        for (int j = 0; j < N; ++j) {
          pfv<64>(in.C, t, r * N + j);
          if (hr) pfv<64>(in.C, t + 1, r * N + j);
        }
      }
    }
  } else if (!SIN) {
#pragma unroll
    for (int i = 0; i < N; ++i) {
#pragma unroll
      for (int j = i; j < N; ++j) pfv<64>(in.ent, t, EN::C + i * N + j);
      pfv<64>(in.ent, t, EN::y + i);
    }
  }
  // row prefetch schedule (distance PD rows): stage 1 streams El/Er/e of
  // t+1, pass B Er of t, pass A Er/El/e of t.
  constexpr int PD = KS_PF_ROWS;
  auto pfE = [&](int i, int64_t c) {
    if (!L0 && !SIN) pfv<64>(in.ent, c, EN::e + i);
    else if (L0 && !CE) pfv<64>(in.e, c, i);
  };
#pragma unroll
  for (int i = 0; i < PD; ++i) {
    if (hr) {
      pfEl(i, t + 1);
      pfEr(i, t + 1);
      pfE(i, t + 1);
    } else if (hl) {
      pfEr(i, t);
    }
  }
  if (!r0) {
  } else if (!L0) {
#pragma unroll
    for (int i = 0; i < N; ++i) {
#pragma unroll
      for (int j = i; j < N; ++j) R[TR::at(i, j)] = ldC(i * N + j, t);
      z[i] = ldY(i, t);
    }
  } else {
#pragma unroll
    for (int i = 0; i < N; ++i)
#pragma unroll
      for (int j = i; j < N; ++j) R[TR::at(i, j)] = (j == i) ? kEmptyRow : 0.0;
#pragma unroll UR
    for (int r = 0; r < in.RC; ++r) {
      double row[N];
#pragma unroll
      for (int j = 0; j < N; ++j) row[j] = ldC(r * N + j, t);
      double yr = ldY(r, t);
      stream_row(R, z, row, yr, 1.0);
    }
  }

  // ---- stage 1: rows of [El_{t+1} | Er_{t+1} | e_{t+1}] into [R | X | z] ----
  // leftover rows [0 | d | y~] (rows of D~_{t+1}) are parked, with their
  // weights, for stage 3.
  if (r0 && hr) {
    const int64_t u = t + 1;
#pragma unroll UR
    for (int i = 0; i < N; ++i) {
      double el[N], er[N];
#pragma unroll
      for (int j = 0; j < N; ++j) {
        el[j] = ldEl(i * N + j, u);
        er[j] = ldEr(i * N + j, u);
      }
      double ee = ldE(i, u);
      if (i + PD < N) {
        pfEl(i + PD, u);
        pfEr(i + PD, u);
        pfE(i + PD, u);
      } else if (hl) {
        pfEr(i + PD - N, t);
      }
      double wl = 1.0;
      rot_row<N>(R, el, wl, [&](int k, double yk, double sb) {
#pragma unroll
        for (int j = 0; j < N; ++j) gapp(X[k][j], er[j], yk, sb);
        gapp(z[k], ee, yk, sb);
      });
#pragma unroll
      for (int j = 0; j < N; ++j) park(kLeft + i * (N + 2) + j, er[j]);
      park(kLeft + i * (N + 2) + N, ee);
      park(kLeft + i * (N + 2) + N + 1, wl);
    }
  }

  // ---- stage 2, pass B: rows of [Er_t | 0] into [R~_t | X_t] -> R_tt, R_{t,t+1}, X~_t ----
  // (pass A below recomputes the same rotations -- bitwise, same inputs and
  // operations -- for [El_t | e_t]).
  if (r0) {
#pragma unroll
    for (int k = 0; k < TR::size; ++k) park(kRt + k, R[k]);
    if (SPL) {   // z~_t for pass A's thread
#pragma unroll
      for (int i = 0; i < N; ++i) park(kParkDoubles<N> + i, z[i]);
    }
  }
  split_bar(1);
  if (r0 && !L0 && !SIN && hr) {   // stage 3's base block C_{t+1}, y_{t+1}
#pragma unroll
    for (int i = 0; i < N; ++i) {
#pragma unroll
      for (int j = i; j < N; ++j) pfv<64>(in.ent, t + 1, EN::C + i * N + j);
      pfv<64>(in.ent, t + 1, EN::y + i);
    }
  }
  if (!r0) {
  } else if (hl) {
#pragma unroll UR
    for (int i = 0; i < N; ++i) {
      double er[N], xr[N];
#pragma unroll
      for (int j = 0; j < N; ++j) {
        er[j] = ldEr(i * N + j, t);
        xr[j] = 0.0;
      }
      if (i + PD < N) pfEr(i + PD, t);
      else {
        pfEr(i + PD - N, t);
        pfEl(i + PD - N, t);
        pfE(i + PD - N, t);
      }
      double wl = 1.0;
      rot_row<N>(R, er, wl, [&](int k, double yk, double sb) {
#pragma unroll
        for (int j = 0; j < N; ++j) gapp(X[k][j], xr[j], yk, sb);
      });
      if (hr) {
        const double w = wscale(wl);
#pragma unroll
        for (int j = 0; j < N; ++j) sto(EN::Er + i * N + j, w * xr[j]);   // X~_t
      }
    }
  } else if (hr) {
#pragma unroll UR
    for (int i = 0; i < N; ++i) {
#pragma unroll
      for (int j = 0; j < N; ++j) sto(EN::Er + i * N + j, 0.0);
    }
  }
  // T_r = R_tt^{-1} R_{t,t+1} = U^{-1} X (unit triangular: no division)
  if (r0) {
#pragma unroll
    for (int i = N - 1; i >= 0; --i) {
#pragma unroll
      for (int c = 0; c < N; ++c) {
        double sr = X[i][c];
#pragma unroll
        for (int k = i + 1; k < N; ++k) sr = fma(-R[TR::at(i, k)], X[k][c], sr);
        X[i][c] = sr;
      }
    }
#pragma unroll
    for (int i = 0; i < N; ++i)
#pragma unroll
      for (int j = 0; j < N; ++j) str(RR::Tr + i * N + j, X[i][j]);
  }

  // ---- stage 3: [D~_{t+1}; C_{t+1}; Zs] -> the survivor's C'_{t+1}, y' ----
  if (r1 && hr) {
    const int64_t u = t + 1;
    double R3[TR::size];
    double z3[N];
    if (!L0) {
#pragma unroll
      for (int i = 0; i < N; ++i) {
#pragma unroll
        for (int j = i; j < N; ++j) R3[TR::at(i, j)] = ldC(i * N + j, u);
        z3[i] = ldY(i, u);
      }
    } else {
#pragma unroll
      for (int i = 0; i < N; ++i)
#pragma unroll
        for (int j = i; j < N; ++j) R3[TR::at(i, j)] = (j == i) ? kEmptyRow : 0.0;
#pragma unroll
      for (int i = 0; i < N; ++i) z3[i] = 0.0;
#pragma unroll UR
      for (int r = 0; r < in.RC; ++r) {
        double row[N];
#pragma unroll
        for (int j = 0; j < N; ++j) row[j] = ldC(r * N + j, u);
        double yr = ldY(r, u);
        stream_row(R3, z3, row, yr, 1.0);
      }
    }
    const int nrows = zs_in ? 2 * N : N;    // leftover rows, then the odd level's Zs (reading R5)
#pragma unroll UR
    for (int i = 0; i < nrows; ++i) {
      double row[N], zr, wl;
      if (i < N) {
#pragma unroll
        for (int j = 0; j < N; ++j) row[j] = unpark(kLeft + i * (N + 2) + j);
        zr = unpark(kLeft + i * (N + 2) + N);
        wl = unpark(kLeft + i * (N + 2) + N + 1);
        if (L0 && wl > kConsumed) continue;   // consumed in stage 1: no D~ row
      } else {
        if (ZS && zsync && i == N) {   // the odd level's last column runs in another thread
          while (*zsync != zval) {
          }
          __threadfence_block();
        }
#pragma unroll
        for (int j = 0; j < N; ++j) row[j] = zs_[(i - N) * (N + 1) + j];
        zr = zs_[(i - N) * (N + 1) + N];
        wl = 1.0;
      }
      stream_row(R3, z3, row, zr, wl);
    }
    // (rho, U) in the upper triangle; the lower triangle is never read.  The
    // multi-GPU boundary entry (OAOS: AoS layout) has the same form: the
    // boundary system runs on these kernels too (SURVEY §8(e) invariant).
#pragma unroll
    for (int i = 0; i < N; ++i) {
#pragma unroll
      for (int j = i; j < N; ++j) sto(EN::C + i * N + j, R3[TR::at(i, j)]);
      sto(EN::y + i, z3[i]);
    }
    sto(EN::nrm, sqrt(ref2u));
  }

  // ---- stage 2, pass A: rows of [Er_t | El_t | e_t] into [R~_t | 0 | z~_t] ----
  if (r2) {   // (SPL) roles 0 and 1 are done
#pragma unroll
  for (int k = 0; k < TR::size; ++k) R[k] = unpark(kRt + k);
  if (SPL) {
#pragma unroll
    for (int i = 0; i < N; ++i) z[i] = unpark(kParkDoubles<N> + i);
  }
  double Rl[N][N];
#pragma unroll
  for (int i = 0; i < N; ++i)
#pragma unroll
    for (int j = 0; j < N; ++j) Rl[i][j] = 0.0;
  if (hl) {
#pragma unroll UR
    for (int i = 0; i < N; ++i) {
      double er[N], el[N];
#pragma unroll
      for (int j = 0; j < N; ++j) {
        er[j] = ldEr(i * N + j, t);
        el[j] = ldEl(i * N + j, t);
      }
      double ee = ldE(i, t);
      if (i + PD < N) {
        pfEr(i + PD, t);
        pfEl(i + PD, t);
        pfE(i + PD, t);
      }
      double wl = 1.0;
      rot_row<N>(R, er, wl, [&](int k, double yk, double sb) {
#pragma unroll
        for (int j = 0; j < N; ++j) gapp(Rl[k][j], el[j], yk, sb);
        gapp(z[k], ee, yk, sb);
      });
      if (hr || zs_out) {
        const double w = wscale(wl);
        if (hr) {
#pragma unroll
          for (int j = 0; j < N; ++j) sto(EN::El + i * N + j, w * el[j]);   // Z_t
          sto(EN::e + i, w * ee);                                           // z^_t
        } else {
#pragma unroll
          for (int j = 0; j < N; ++j) zs_[i * (N + 1) + j] = w * el[j];
          zs_[i * (N + 1) + N] = w * ee;
        }
      }
    }
  } else if (hr) {
#pragma unroll UR
    for (int i = 0; i < N; ++i) {
#pragma unroll
      for (int j = 0; j < N; ++j) sto(EN::El + i * N + j, 0.0);
      sto(EN::e + i, 0.0);
    }
  }
  if (ZS && zs_out && zsync) {   // Z rows published to the last pair's thread
    __threadfence_block();
    *zsync = zval;
  }

  // ---- post: rank check, T_l = U^{-1} Rl, w = U^{-1} z, P = U^{-1} D^{-1} U^{-T} ----
  {
    const double thr = kRankTol * kRankTol * ref2;   // |R_kk|^2 = d_k = 1/rho_k vs (tol |col|)^2
    bool bad = false;
#pragma unroll
    for (int d = 0; d < N; ++d) bad |= !(R[TR::at(d, d)] * thr < 1.0);
    if (bad) report(a.status, (((t + 1) << (a.level - a.lbase)) - 1) + a.step0, kBadRank);
  }
  double inv[N];   // 1/d_k
#pragma unroll
  for (int i = 0; i < N; ++i) inv[i] = R[TR::at(i, i)];
#pragma unroll
  for (int i = N - 1; i >= 0; --i) {
#pragma unroll
    for (int c = 0; c < N; ++c) {
      double sl = Rl[i][c];
#pragma unroll
      for (int k = i + 1; k < N; ++k) sl = fma(-R[TR::at(i, k)], Rl[k][c], sl);
      Rl[i][c] = sl;
    }
    double sz = z[i];
#pragma unroll
    for (int k = i + 1; k < N; ++k) sz = fma(-R[TR::at(i, k)], z[k], sz);
    z[i] = sz;
  }
#pragma unroll
  for (int i = 0; i < N; ++i) {
#pragma unroll
    for (int j = 0; j < N; ++j) str(RR::Tl + i * N + j, Rl[i][j]);
    str(RR::w + i, z[i]);
  }
  // V = U^{-1} (unit upper, in place of U): V(i,j) = -sum_{k=i+1..j} U(i,k) V(k,j)
#pragma unroll
  for (int i = N - 1; i >= 0; --i) {
#pragma unroll
    for (int j = N - 1; j > i; --j) {
      double s = R[TR::at(i, j)];
#pragma unroll
      for (int k = i + 1; k < j; ++k) s = fma(R[TR::at(i, k)], R[TR::at(k, j)], s);
      R[TR::at(i, j)] = -s;
    }
  }
  // P(i,j) = sum_{k >= j} V(i,k) V(j,k) / d_k   (i <= j, V(k,k) = 1)
#pragma unroll
  for (int i = 0; i < N; ++i) {
#pragma unroll
    for (int j = i; j < N; ++j) {
      double s = 0.0;
#pragma unroll
      for (int k = j; k < N; ++k) {
        const double vik = (k == i) ? 1.0 : R[TR::at(i, k)];
        const double vjk = (k == j) ? 1.0 : R[TR::at(j, k)];
        s = fma(vik, vjk * inv[k], s);
      }
      str(RR::P + TR::at(i, j), s);
    }
  }
  }   // r2
  split_bar(2);
}

// Resident CTAs (of 64 threads) per SM the register allocation targets.
// n = 6, level 0 with a constant (stride-0) observation model: every block but
// o is staged in shared memory, so a register cap for 6 CTAs/SM (168
// registers, 104 bytes of stack) pays there (c5 factor L0 0.848 -> 0.821 ms;
// 5 CTAs: 0.828) while it slows the levels >= 1 (5 CTAs: L1 0.576 -> 0.747
// ms, 216 bytes of spills).
constexpr int factor_min_blocks(int n, bool l0c = false) {
  return n <= 4 ? 8 : n == 5 ? 7 : n == 6 ? (l0c ? KS_F6_L0C_BLOCKS : KS_F6_BLOCKS) : 4;
}

// One work item of a factor level: pair p (plus, on an odd level, the last
// column without right neighbour, handled first by the last pair's thread).
// split_odd(K, T): on an odd level >= 1 the last column runs in its own thread
// (index K/2, after the pairs) concurrently with the last pair, whose stage 3
// waits for its Z rows on the shared-memory word zsync (value zval) -- when
// that thread is in the same CTA of T threads as the last pair's (the odd
// level then costs one pair elimination, not two in series).  The fused tail
// keeps the serial form (the larger ZS body costs it more I-cache than the
// split saves at n = 6).
__host__ __device__ inline bool split_odd(int64_t K, int T) { return K >= 3 && (K & 1) && ((K / 2) % T) != 0; }
template <int N, bool L0, bool CE, bool CC, bool OAOS, bool SIN = false, bool ZS = false>
__device__ __forceinline__ void factor_item(const SmallFactorArgs &a, int64_t p, volatile int *zsync = nullptr,
                                            int zval = 0) {
  if (!ZS) zsync = nullptr;   // ZS: compiled with the split-odd-level code
  const int64_t K = a.K;
  const bool single_only = (K == 1);
  // split odd level (zsync): thread K/2 eliminates the last column, the last
  // pair waits for its Z rows; else the last pair's thread does both
  const bool lastcol = zsync && p == K / 2;
  const bool triple = !zsync && (K >= 3) && (K & 1) && (p == K / 2 - 1);
  const bool waits = zsync && (p == K / 2 - 1);
  // pass 0: the odd level's last column (no right neighbour), pass 1: the pair.
  // One inlined call site per pass keeps the (large, fully unrolled) body at
  // most twice in the instruction cache.
#pragma unroll 1
  for (int pass = (single_only || triple || lastcol) ? 0 : 1; pass < ((single_only || lastcol) ? 1 : 2); ++pass) {
    const int64_t t = pass == 0 ? K - 1 : 2 * p;
    const bool hl = t + a.t0 > 0;
    if (pass == 0)
      small_eliminate<N, L0, CE, CC, OAOS, SIN, ZS>(a, t, false, hl, 0, false, hl, zsync, zval);
    else
      small_eliminate<N, L0, CE, CC, OAOS, SIN, ZS>(a, t, true, hl, p, (triple || waits) && (K - 1 + a.t0 > 0),
                                                    false, waits ? zsync : nullptr, zval);
  }
}

// The fused tail's split form (small_eliminate SPL): slot `slot` (0..63) of
// role `role`; three threads per pair.  Every thread makes the same calls
// (the barriers inside): an odd level (serial form: the last pair's slot
// eliminates the last column first) has a round 0 in which only that slot
// works; the base case (K = 1) is slot 0's single column.
template <int N, bool SIN = true, bool OAOS = false>
__device__ __forceinline__ void factor_item_split(const SmallFactorArgs &a, int64_t p, bool has, int role, int slot) {
  const int64_t K = a.K;
  if (K == 1) {
    const bool hl = a.t0 > 0;
    small_eliminate<N, false, false, false, OAOS, SIN, false, true>(a, 0, false, hl, 0, false, hl, nullptr, 0, role,
                                                                       slot, has);
    return;
  }
  const bool odd = (K >= 3) && (K & 1);
  if (odd) {
    const int64_t t = K - 1;
    const bool hl = t + a.t0 > 0;
    small_eliminate<N, false, false, false, OAOS, SIN, false, true>(a, t, false, hl, 0, false, hl, nullptr, 0, role,
                                                                       slot, has && p == K / 2 - 1);
  }
  const int64_t t = 2 * p;
  const bool hl = t + a.t0 > 0;
  const bool triple = odd && p == K / 2 - 1;
  small_eliminate<N, false, false, false, OAOS, SIN, false, true>(
      a, t, true, hl, p, triple && (K - 1 + a.t0 > 0), false, nullptr, 0, role, slot, has);
}

// A level >= 1 with few pairs (latency-bound: at most one 64-pair CTA per
// SM) in the split form: 192 threads = three roles x 64 pair slots per CTA,
// the odd level's last column in the serial form (its slot's round 0).
template <int N, bool OAOS>
__global__ void __launch_bounds__(kTailThreads, 1) small_factor_split_kernel(SmallFactorArgs a) {
  const int slot = threadIdx.x & 63, role = threadIdx.x >> 6;
  const int64_t npairs = a.K >= 2 ? a.K / 2 : 1;
  const int64_t p = (int64_t)blockIdx.x * 64 + slot;
  factor_item_split<N, false, OAOS>(a, p, p < npairs, role, slot);
}

template <int N, bool L0, bool CE, bool CC, bool OAOS, bool ZS = false>
__global__ void __launch_bounds__(64, factor_min_blocks(N, L0 && CC)) small_factor_kernel(SmallFactorArgs a) {
  if (L0 && (CE || CC)) {   // stage the constant (stride-0) level-0 blocks once per CTA
    extern __shared__ double smem_park[];
    double *cst = smem_park + (size_t)blockDim.x * kParkDoubles<N>;
    for (int k = threadIdx.x; k < CstOff<N>::size; k += blockDim.x) {
      double v = 0.0;
      if (CE && k < CstOff<N>::e + N) {
        v = k < CstOff<N>::Er ? a.in.El.p[k] : k < CstOff<N>::e ? a.in.Er.p[k - CstOff<N>::Er]
                                                              : a.in.e.p[k - CstOff<N>::e];
      } else if (CC && k >= CstOff<N>::C && k - CstOff<N>::C < a.in.RC * N) {
        v = a.in.C.p[k - CstOff<N>::C];
      } else if (CC && a.in.yfuse && k >= CstOff<N>::Mi) {
        const int r = (k - CstOff<N>::Mi) / kSmallMaxM, q = (k - CstOff<N>::Mi) % kSmallMaxM;
        v = (r < a.in.RC && q < a.in.RC) ? a.in.Minv[r * a.in.RC + q] : 0.0;
      }
      cst[k] = v;
    }
    __syncthreads();
  }
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t npairs = a.K >= 2 ? a.K / 2 : 1;
  if constexpr (ZS) {   // launched only when split_odd(K, 64)
    __shared__ int zsync;
    if (threadIdx.x == 0) zsync = 0;
    __syncthreads();
    if (p > npairs) return;
    factor_item<N, L0, CE, CC, OAOS, false, true>(a, p, &zsync, 1);
    return;
  }
  if (p >= npairs) return;
  factor_item<N, L0, CE, CC, OAOS>(a, p);
}

// The recursion's tail: every level from the first one
// with K <= tail_max_cols<N>() up to the base case in ONE CTA and one launch.
// The level entries live in shared memory (ping-pong buffers: level L reads
// one, writes the other, K halves every level), so the tail pays neither a
// launch nor an L2/DRAM round trip per level -- only the latency of one pair
// elimination per level.  R records go to HBM as usual (the backward reads
// them).  Same per-column code (small_eliminate) as the level kernels.
// shared memory of the tail kernel with first-level width K0 (a multiple of
// 64): park | const | buffer A (K0 columns) | buffer B (max(64, K0 / 2))
template <int N>
__host__ __device__ constexpr size_t tail_smem_doubles(int K0) {
  return (size_t)64 * kParkSP<N> + CstOff<N>::size +
         (size_t)(K0 + (K0 / 2 > 64 ? K0 / 2 : 64)) * (3 * N * N + 2 * N + 1);
}
template <int N>
__host__ __device__ constexpr int tail_max_cols() {
  return tail_smem_doubles<N>(128) * 8 <= 227 * 1024 ? 128 : tail_smem_doubles<N>(64) * 8 <= 227 * 1024 ? 64 : 0;
}
template <int N>
__host__ __device__ constexpr size_t tail_smem_bytes() {
  return tail_max_cols<N>() ? tail_smem_doubles<N>(tail_max_cols<N>()) * sizeof(double) : 0;
}
template <int N>
__global__ void __launch_bounds__(kTailThreads, 1) small_factor_tail_kernel(SmallTailArgs t) {
  extern __shared__ double smem_park[];
  constexpr int64_t E = 3 * N * N + 2 * N + 1;
  double *bufA = smem_park + (size_t)64 * kParkSP<N> + CstOff<N>::size;
  // W == 0: one CTA runs whole levels; W > 0: CTA c owns the subtree of the W
  // columns [cW, cW + W) of the first level (W a power of two, every level
  // halving exactly), so all its levels are local (a column's
  // left neighbour in another subtree is only a target of blocks stored here)
  const int64_t c = blockIdx.x;
  const int64_t K0 = t.W ? t.W : t.K[0];
  double *bufB = bufA + ptiled_doubles(K0, E);
  {   // first-level entries: global (written by the last level kernel) -> buffer A
    const int64_t cnt = ptiled_doubles(K0, E);
    const double *src = t.ent0 + (t.W ? c * t.W * E : 0);
    for (int64_t i = threadIdx.x; i < cnt; i += blockDim.x) bufA[i] = src[i];
  }
  __syncthreads();
  double *in = bufA, *out = bufB;
  for (int lv = 0; lv < t.nlev; ++lv) {
    SmallFactorArgs a = t.base;
    a.K = t.K[lv];
    a.level = t.level[lv];
    a.rec = t.rec[lv];
    a.in.ent = TView{in, 64 * E};
    const int64_t kloc = t.W ? (t.W >> lv) : a.K;            // this CTA's columns
    a.ent_off = t.W ? c * kloc : 0;
    const bool last = lv + 1 == t.nlev;
    a.out = last ? t.out_last : TView{out, 64 * E};
    a.outAoS = last ? t.out_last_aos : 0;
    a.out_off = (t.W && !last) ? c * (kloc / 2) : 0;
    const int64_t npairs = t.W ? kloc / 2 : (a.K >= 2 ? a.K / 2 : 1);   // <= 64
    const int slot = threadIdx.x & 63, role = threadIdx.x >> 6;
    factor_item_split<N>(a, (t.W ? c * (kloc / 2) : 0) + slot, slot < npairs, role, slot);
    __syncthreads();
    double *tmp = in;
    in = out;
    out = tmp;
  }
}

// -------------------------------------------------------------- backward ---

// One thread per eliminated column t of level L (P:592-600 and Alg. 2,
// P:792-824):
//   x_t    = w - T_l x_l - T_r x_r
//   S_tl   = -(T_l S_ll + T_r S_lr^T),  S_tr = -(T_l S_lr + T_r S_rr)   (S_{t,I} = -T S_II)
//   S_tt   = P - S_tl T_l^T - S_tr T_r^T  (upper triangle computed, mirrored)
// S_lr = S_{t-1,t+1} is the level-(L+1) cross block; S_{t-1,t} = S_tl^T and
// S_{t,t+1} = S_tr are stored for level L-1.  With do_state and do_cov both
// set, one pass over the R records serves the solve and SelInv
// (ks_solve_selinv).
// Backward CTA: BC eliminated columns (one record tile), two threads per
// column (warp 0: the "left" half of Alg. 2's products, warp 1: the "right").
constexpr int kBwdCols = 32;
// resident CTAs per SM the register allocation targets (no spills at n = 6..8)
#ifndef KS_BWD6_BLOCKS
#define KS_BWD6_BLOCKS 4
#endif
constexpr int bwd_min_blocks(int n) { return n <= 5 ? 5 : n == 6 ? KS_BWD6_BLOCKS : 3; }
template <int N>
__host__ __device__ constexpr int rs_doubles() { return 2 * N * N + N + N * (N + 1) / 2; }
// S_tt staging row: NN doubles padded to a multiple of 2 (16-byte rows for
// the bulk store) and to an odd number of 16-byte units (fewer bank conflicts)
template <int N>
__host__ __device__ constexpr int bwd_sp() { return ((N * N + 1) / 2) % 2 ? 2 * ((N * N + 1) / 2) : 2 * ((N * N + 1) / 2) + 2; }
// shared memory: record tile [RS][BC] | S_lr tile [NN][BC] | max(neighbour
// blocks [NN][BC+1], Q_l, Q_r [2][NT][BC+1]); the S_tt staging rows [BC][SP]
// overlay the record tile's T_l, T_r part (dead once Q_l, Q_r are formed)
template <int N>
__host__ __device__ constexpr size_t bwd_smem_doubles() {
  return (size_t)kBwdCols * (rs_doubles<N>() + N * N) +
         ((size_t)N * N > (size_t)N * (N + 1) ? (size_t)N * N : (size_t)N * (N + 1)) * (kBwdCols + 1);
}
static_assert(bwd_sp<1>() <= 2 && bwd_sp<6>() <= 72 && bwd_sp<8>() <= 128, "S_tt staging must fit in T_l, T_r");

// 8-byte asynchronous global -> shared copy (LDGSTS); src_size 0 zero-fills.
__device__ __forceinline__ void cp_async8(double *sdst, const double *gsrc, bool valid) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(sdst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(sa), "l"(gsrc), "r"(valid ? 8 : 0));
}

// mbarrier + 1-D bulk copy (the TMA engine: UBLKCP in SASS) of a contiguous
// global range into shared memory.
__device__ __forceinline__ unsigned smem_u32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long *bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long *bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, unsigned bytes, unsigned long long *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long *bar, unsigned phase) {
  asm volatile(
      "{\n"
      " .reg .pred p;\n"
      "KS_MBAR_WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra KS_MBAR_WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}

// One tile of eliminated columns (32 columns, 64 threads: see the kernel
// below).  TAIL: called once per level by the fused backward tail kernel --
// the mbarrier is initialised by the caller and reused (phase bit), S_tt goes
// out with plain stores (the next level of the same kernel reads it), and a
// tile index beyond the level only takes part in the CTA barriers.
template <int N, bool TAIL>
__device__ __forceinline__ void bwd_tile(const SmallBackwardArgs &a, int64_t tile, int tid, double *bsm,
                                         unsigned long long *mbarp, unsigned phase, int64_t bbeg = 0,
                                         int64_t bend = INT64_MAX) {
  using TR = Tri<N>;
  using RR = Rr<N>;
  constexpr int NN = N * N, BC = kBwdCols, NB = BC + 1, RS = rs_doubles<N>(), SP = bwd_sp<N>(),
                NT = N * (N + 1) / 2;
  const int col = tid & (BC - 1);
  const bool right = tid >= BC;      // warp-uniform
  const int64_t b0 = tile * BC, b = b0 + col, t = 2 * b;
  const bool tile_live = b0 < (a.K + 1) / 2;
  // columns outside [bbeg, bend) belong to another CTA's subtree: staged
  // (harmless) but neither computed nor written
  const bool active = t < a.K && b >= bbeg && b < bend;
  const bool hl = (t + a.t0) > 0, hr = (t + 1) < a.K;
  const int64_t step = 1ll << a.shift;
  const int64_t j = ((t + 1) << a.shift) - 1, jl = j - step, jr = j + step;
  double xl[N], xr[N];
  // the state x_t: the left thread of a column in the solve-only path, the
  // right one (the half with less SelInv work) when both are computed
  const bool xside = a.do_cov ? right : !right;
  if (a.do_state && active && xside) {
    const double *pl = hl ? (jl < 0 ? a.xhalo : a.x + jl * N) : nullptr;
    const double *pr = hr ? a.x + jr * N : nullptr;
#pragma unroll
    for (int k = 0; k < N; ++k) {
      xl[k] = pl ? pl[k] : 0.0;
      xr[k] = pr ? pr[k] : 0.0;
    }
  }
  if (!a.do_cov) {   // solve only: direct coalesced record loads, no staging
    if (!active || right) return;
#pragma unroll
    for (int i = 0; i < N; ++i) {
      double s = ldv<32>(a.rec, b, RR::w + i);
#pragma unroll
      for (int k = 0; k < N; ++k) {
        s = fma(-ldv<32>(a.rec, b, RR::Tl + i * N + k), xl[k], s);
        s = fma(-ldv<32>(a.rec, b, RR::Tr + i * N + k), xr[k], s);
      }
      a.x[j * N + i] = s;
    }
    return;
  }

  // Staging.  (1) The CTA's R records are one tile of the tiled record array
  // (32 columns x RS doubles, contiguous) and its cross blocks S_lr one tile
  // of the tiled level-(L+1) cross array: two bulk copies by the TMA engine,
  // completion on an mbarrier.  (2) The 33 distinct neighbour covariance
  // blocks of the CTA's 32 columns (level-(L+1) columns b0-1 .. b0+31, each a
  // contiguous n^2 block of S in step order), strided in HBM: cp.async,
  // element-major in shared memory.  (3) The neighbour states go straight
  // to registers, issued before the waits.
  // Alg. 2's products are split between the two threads of a column:
  //   left:  S_tl = -(T_l S_ll + T_r S_lr^T),  Q_l = S_tl T_l^T, x_t
  //   right: S_tr = -(T_l S_lr + T_r S_rr),    Q_r = S_tr T_r^T
  // and S_tt = P + Q_l + Q_r (upper triangle, mirrored) goes back through
  // shared memory as one bulk store per column.
  double *REC = bsm;                 // [RS][32]
  double *SLR = bsm + BC * RS;       // [NN][32]   the tile of the tiled S_lr array
  double *Snb = SLR + BC * NN;       // [NN][NB]   (later: Q_l, Q_r [2][NT][NB])
  const bool xs = a.Xup.p != nullptr;
  if (tid == 0 && tile_live) {
    if (!TAIL) mbar_init(mbarp, 1);
    mbar_expect_tx(mbarp, (unsigned)((RS + (xs ? NN : 0)) * 32 * 8));
    bulk_g2s(REC, a.rec.p + tile * a.rec.ts, (unsigned)(RS * 32 * 8), mbarp);
    if (xs) bulk_g2s(SLR, a.Xup.p + tile * a.Xup.ts, (unsigned)(NN * 32 * 8), mbarp);
  }
  const int64_t Kup = a.K / 2;       // columns of level L+1
  {
    // neighbour block sblk = tid (0..32) of the CTA, thread tid stages it
    const int sblk = tid;
    if (sblk <= BC) {
      const int64_t q = b0 - 1 + sblk;
      const double *src = nullptr;
      if (q == -1) {
        if (a.t0 > 0) src = a.Shalo;
      } else if (q >= 0 && q < Kup) {
        src = a.S + (((q + 1) << (a.shift + 1)) - 1) * NN;
      }
      const bool ok = src != nullptr;
      const double *s0 = ok ? src : a.S;
#pragma unroll
      for (int e = 0; e < NN; ++e) cp_async8(&Snb[e * NB + sblk], s0 + (ok ? e : 0), ok);
    }
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
  __syncthreads();                   // mbarrier init visible; neighbour blocks landed
  if (tile_live) mbar_wait(mbarp, phase);
  const double *myrec = REC + col;
  auto rec = [&](int e) { return myrec[e * 32]; };
  if (active && a.do_state && xside) {
#pragma unroll
    for (int i = 0; i < N; ++i) {
      double s = rec(RR::w + i);
#pragma unroll
      for (int k = 0; k < N; ++k) {
        s = fma(-rec(RR::Tl + i * N + k), xl[k], s);
        s = fma(-rec(RR::Tr + i * N + k), xr[k], s);
      }
      a.x[j * N + i] = s;
    }
  }
  double Slr[N][N];
#pragma unroll
  for (int r = 0; r < N; ++r)
#pragma unroll
    for (int c = 0; c < N; ++c) Slr[r][c] = (hl && hr) ? SLR[(r * N + c) * BC + col] : 0.0;
  double Sd[TR::size];               // left: S_ll, right: S_rr
  if (active) {
#pragma unroll
    for (int r = 0; r < N; ++r)
#pragma unroll
      for (int c = r; c < N; ++c) Sd[TR::at(r, c)] = Snb[(r * N + c) * NB + col + (right ? 1 : 0)];
  }
  __syncthreads();                   // Snb is dead: its space becomes Q_l, Q_r
  double *Qs = Snb + (right ? NT * NB : 0) + col;   // this side's Q [NT][NB]
  double *Stt = REC + col * SP;      // over T_l, T_r (after the Q barrier)
  if (active) {
    // one code path per side (warp-uniform branch), so neither side executes
    // the other's products
    auto side = [&](auto right_c) {
      constexpr bool RIGHT = decltype(right_c)::value;
      // the T block this side multiplies from the right: T_l (left) / T_r (right)
      constexpr int TO = RIGHT ? RR::Tr : RR::Tl;
#pragma unroll(N <= 6 ? N : 1)
      for (int i = 0; i < N; ++i) {
        double tl[N], tr[N], A[N];
#pragma unroll
        for (int k = 0; k < N; ++k) {
          tl[k] = rec(RR::Tl + i * N + k);
          tr[k] = rec(RR::Tr + i * N + k);
        }
#pragma unroll
        for (int c = 0; c < N; ++c) {
          double s = 0.0;
#pragma unroll
          for (int k = 0; k < N; ++k) {
            const double sd = k <= c ? Sd[TR::at(k, c)] : Sd[TR::at(c, k)];
            if (!RIGHT) {            // S_tl = -(T_l S_ll + T_r S_lr^T)
              s = fma(tl[k], sd, s);
              s = fma(tr[k], Slr[c][k], s);
            } else {                 // S_tr = -(T_l S_lr + T_r S_rr)
              s = fma(tl[k], Slr[k][c], s);
              s = fma(tr[k], sd, s);
            }
          }
          A[c] = -s;
        }
        if (a.Xcur.p) {
#pragma unroll
          for (int c = 0; c < N; ++c) {
            if (!RIGHT && hl) stv<32>(a.Xcur, t, c * N + i, A[c]);      // slot t-1: S_{t-1,t} = S_tl^T
            if (RIGHT && hr) stv<32>(a.Xcur, t + 1, i * N + c, A[c]);   // slot t:   S_{t,t+1} = S_tr
          }
        }
        // row i of Q = S_t* T_*^T (upper part jj >= i); the jj chains are independent
#pragma unroll
        for (int jj = 0; jj < N; ++jj) {
          if (jj < i) continue;
          double q = 0.0;
#pragma unroll
          for (int k = 0; k < N; ++k) q = fma(A[k], rec(TO + jj * N + k), q);
          Qs[(i * N - (i * (i - 1)) / 2 + (jj - i)) * NB] = q;
        }
      }
    };
    if (right) side(std::true_type{});
    else side(std::false_type{});
  }
  __syncthreads();
  if (active) {
    // S_tt = P - S_tl T_l^T - S_tr T_r^T = P - Q_l - Q_r (upper part,
    // mirrored), the upper-triangle entries split between the two threads
    constexpr int ES = (NT + 1) / 2;
    const double *Q0 = Snb + col;    // Q_l [NT][NB] then Q_r [NT][NB]
#pragma unroll
    for (int i = 0; i < N; ++i)
#pragma unroll
      for (int jj = i; jj < N; ++jj) {
        const int e = TR::at(i, jj);
        if ((e < ES) != right) {
          const double sv = (rec(RR::P + e) - Q0[e * NB]) - Q0[(NT + e) * NB];
          Stt[i * N + jj] = sv;
          Stt[jj * N + i] = sv;
        }
      }
    // generic-proxy writes made visible to the bulk (async-proxy) copies
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();
  if (active && !right) {
    if constexpr (TAIL || NN % 2 != 0) {
#pragma unroll
      for (int e = 0; e < NN; ++e) a.S[j * NN + e] = Stt[e];
    } else {   // 16-byte multiple and alignment: one bulk store
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(a.S + j * NN),
                   "r"(smem_u32(Stt)), "r"((unsigned)(NN * 8))
                   : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    }
  }
}


template <int N>
__global__ void __launch_bounds__(2 * kBwdCols, bwd_min_blocks(N)) small_backward_kernel(SmallBackwardArgs a) {
  extern __shared__ __align__(16) double bsm[];
  __shared__ __align__(8) unsigned long long mbar;
  bwd_tile<N, false>(a, blockIdx.x, threadIdx.x, bsm, &mbar, 0);
}

// The backward of the recursion's tail (the levels the fused factor tail ran)
// in one CTA and one launch, top level first: two tiles (4 warps) per round,
// a CTA barrier between levels (each level reads what the one above wrote).
template <int N>
__global__ void __launch_bounds__(4 * kBwdCols, 1) small_backward_tail_kernel(SmallBwdTailArgs t) {
  extern __shared__ __align__(16) double bsm[];
  __shared__ __align__(8) unsigned long long mbar[2];
  const int half = threadIdx.x / (2 * kBwdCols), tid = threadIdx.x % (2 * kBwdCols);
  double *my = bsm + half * bwd_smem_doubles<N>();
  if (tid == 0) mbar_init(&mbar[half], 1);
  __syncthreads();
  unsigned phase = 0;
  const int64_t c = blockIdx.x;
  for (int lv = 0; lv < t.nlev; ++lv) {
    SmallBackwardArgs a = t.base;
    a.rec = t.rec[lv];
    a.K = t.K[lv];
    a.shift = t.shift[lv];
    a.Xup = t.Xup[lv];
    a.Xcur = t.Xcur[lv];
    // W == 0: the whole level; else this CTA's subtree (W columns at the
    // bottom level, W >> (nlev-1-lv) at this one): eliminated columns
    // [bbeg, bend), inside one or more 32-column record tiles
    int64_t bbeg = 0, bend = (a.K + 1) / 2;
    if (t.W) {
      const int64_t ne = (t.W >> (t.nlev - 1 - lv)) / 2;
      bbeg = c * ne;
      bend = bbeg + ne;
    }
    const int64_t tb = bbeg / kBwdCols, te = (bend + kBwdCols - 1) / kBwdCols;
    for (int64_t r = 0; tb + 2 * r < te; ++r) {
      const int64_t tile = tb + 2 * r + half;
      const bool live = tile < te;
      bwd_tile<N, true>(a, live ? tile : ((a.K + 1) / 2 + kBwdCols) / kBwdCols, tid, my, &mbar[half], phase, bbeg,
                        bend);
      if (live && tile * kBwdCols < (a.K + 1) / 2) phase ^= 1u;
      __syncthreads();
    }
  }
}

// ------------------------------------------------ TMA-tensor backward ---
//
// The regular-level fused backward for even n (n^2 and n doubles are 16-byte
// multiples): every strided block of the tile moves as ONE TMA tensor copy.
// In step order the level-(L+1) neighbours q = b0-1 .. b0+31 of the tile's
// columns and the tile's own level-L columns are both rows of a 2-D view of
// S (and x) with row pitch 2^(L+1) blocks, so a [33][n^2] box loads the 33
// neighbour blocks (row -1 out of bounds: zero-filled, patched from the
// shard halo) and a [32][n^2] box stores the 32 S_tt blocks (rows past the
// level end are clipped); the same for the states.  With the record and S_lr
// tiles (bulk copies) the whole tile arrives on one mbarrier and leaves in
// two stores, no per-thread global traffic except the cross blocks.
struct BwdMaps {
  CUtensorMap Sout, Snb, xout, xnb;   // box [32][n^2], [33][n^2], [32][n], [33][n]
};
__host__ __device__ constexpr int rnd16(int d) { return (d + 15) / 16 * 16; }
template <int N>
struct BwdT {
  static constexpr int NN = N * N, NT = N * (N + 1) / 2, BC = kBwdCols, NB = BC + 1, RS = rs_doubles<N>();
  // doubles: REC [RS][32] | SLR [NN][32] | SNB [33][NN] / Q [2][NT][NB] | XNB [33][N] | XST [32][N]
  static constexpr int REC = 0, SLR = REC + RS * BC, SNB = SLR + NN * BC,
                       XNB = SNB + rnd16((BC + 1) * NN > 2 * NT * NB ? (BC + 1) * NN : 2 * NT * NB),
                       XST = XNB + rnd16((BC + 1) * N), total = XST + rnd16(BC * N),
                       // levels >= 1 (KS_BWD_XSTAGE): the 64 cross-block slots 2 b0 .. 2 b0 + 63
                       // of the tile = two tiles of the tiled level-L cross array, one bulk store
                       XCS = total, total_x = XCS + 2 * NN * BC;
};
#ifndef KS_BWD_XSTAGE
#define KS_BWD_XSTAGE 1
#endif
__device__ __forceinline__ void tma_load2d(void *dst, const CUtensorMap *m, int c0, int c1, unsigned long long *bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(dst)),
      "l"(m), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_store2d(const CUtensorMap *m, int c0, int c1, const void *src) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.tile.bulk_group [%0, {%1, %2}], [%3];" ::"l"(m), "r"(c0),
               "r"(c1), "r"(smem_u32(src))
               : "memory");
}

template <int N>
__global__ void __launch_bounds__(2 * kBwdCols, bwd_min_blocks(N))
    small_backward_tma_kernel(const SmallBackwardArgs a, const __grid_constant__ BwdMaps m) {
  using TR = Tri<N>;
  using RR = Rr<N>;
  using L = BwdT<N>;
  constexpr int NN = N * N, BC = kBwdCols, NB = BC + 1, RS = L::RS, NT = L::NT;
  extern __shared__ __align__(128) double tsm[];
  __shared__ __align__(8) unsigned long long mbar;
  double *bsm = tsm;
  const int tid = threadIdx.x, col = tid & (BC - 1);
  const bool right = tid >= BC;      // warp-uniform
  const int64_t b0 = (int64_t)blockIdx.x * BC, b = b0 + col, t = 2 * b;
  const bool active = t < a.K;
  const bool hl = (t + a.t0) > 0, hr = (t + 1) < a.K;
  double *REC = bsm + L::REC, *SLR = bsm + L::SLR, *SNB = bsm + L::SNB, *XNB = bsm + L::XNB, *XST = bsm + L::XST;
  const bool xs = a.Xup.p != nullptr;
  if (tid == 0) {
    mbar_init(&mbar, 1);
    mbar_expect_tx(&mbar, (unsigned)(8 * (RS * BC + (xs ? NN * BC : 0) + (BC + 1) * NN + (a.do_state ? (BC + 1) * N : 0))));
    bulk_g2s(REC, a.rec.p + blockIdx.x * a.rec.ts, (unsigned)(RS * BC * 8), &mbar);
    if (xs) bulk_g2s(SLR, a.Xup.p + blockIdx.x * a.Xup.ts, (unsigned)(NN * BC * 8), &mbar);
    tma_load2d(SNB, &m.Snb, 0, (int)(b0 - 1), &mbar);
    if (a.do_state) tma_load2d(XNB, &m.xnb, 0, (int)(b0 - 1), &mbar);
  }
  __syncthreads();                   // mbarrier initialised
  mbar_wait(&mbar, 0);
  if (b0 == 0 && a.t0 > 0) {         // neighbour q = -1: the shard halo
    for (int e = tid; e < NN; e += 2 * BC) SNB[e] = a.Shalo[e];
    if (a.do_state && tid < N) XNB[tid] = a.xhalo[tid];
    __syncthreads();
  }
  const double *myrec = REC + col;
  auto rec = [&](int e) { return myrec[e * BC]; };
  if (active && a.do_state && right) {   // x_t = w - T_l x_l - T_r x_r
#pragma unroll
    for (int i = 0; i < N; ++i) {
      double sx = rec(RR::w + i);
#pragma unroll
      for (int k = 0; k < N; ++k) {
        sx = fma(-rec(RR::Tl + i * N + k), XNB[col * N + k], sx);
        sx = fma(-rec(RR::Tr + i * N + k), XNB[(col + 1) * N + k], sx);
      }
      XST[col * N + i] = sx;
    }
  }
  double Slr[N][N];
#pragma unroll
  for (int r = 0; r < N; ++r)
#pragma unroll
    for (int c = 0; c < N; ++c) Slr[r][c] = (hl && hr) ? SLR[(r * N + c) * BC + col] : 0.0;
  double Sd[TR::size];               // left: S_ll, right: S_rr
#pragma unroll
  for (int r = 0; r < N; ++r)
#pragma unroll
    for (int c = r; c < N; ++c) Sd[TR::at(r, c)] = SNB[(col + (right ? 1 : 0)) * NN + r * N + c];
  __syncthreads();                   // SNB is dead: its space becomes Q_l, Q_r
  double *Qs = SNB + (right ? NT * NB : 0) + col;
  if (active) {
    auto side = [&](auto right_c) {
      constexpr bool RIGHT = decltype(right_c)::value;
      constexpr int TO = RIGHT ? RR::Tr : RR::Tl;
#pragma unroll(N <= 6 ? N : 1)
      for (int i = 0; i < N; ++i) {
        double tl[N], tr[N], A[N];
#pragma unroll
        for (int k = 0; k < N; ++k) {
          tl[k] = rec(RR::Tl + i * N + k);
          tr[k] = rec(RR::Tr + i * N + k);
        }
#pragma unroll
        for (int c = 0; c < N; ++c) {
          double sacc = 0.0;
#pragma unroll
          for (int k = 0; k < N; ++k) {
            const double sd = k <= c ? Sd[TR::at(k, c)] : Sd[TR::at(c, k)];
            if (!RIGHT) {            // S_tl = -(T_l S_ll + T_r S_lr^T)
              sacc = fma(tl[k], sd, sacc);
              sacc = fma(tr[k], Slr[c][k], sacc);
            } else {                 // S_tr = -(T_l S_lr + T_r S_rr)
              sacc = fma(tl[k], Slr[k][c], sacc);
              sacc = fma(tr[k], sd, sacc);
            }
          }
          A[c] = -sacc;
        }
        if (a.Xcur.p) {
          if (KS_BWD_XSTAGE) {   // slot 2 col (+1): tile col >> 4, position 2 col & 31 (+1)
            double *xs = bsm + L::XCS + (col >> 4) * NN * BC + ((2 * col) & 31) + (RIGHT ? 1 : 0);
#pragma unroll
            for (int c = 0; c < N; ++c) xs[(RIGHT ? i * N + c : c * N + i) * BC] = A[c];
          } else {
#pragma unroll
            for (int c = 0; c < N; ++c) {
              if (!RIGHT && hl) stv<32>(a.Xcur, t, c * N + i, A[c]);      // slot t-1: S_{t-1,t} = S_tl^T
              if (RIGHT && hr) stv<32>(a.Xcur, t + 1, i * N + c, A[c]);   // slot t:   S_{t,t+1} = S_tr
            }
          }
        }
#pragma unroll
        for (int jj = 0; jj < N; ++jj) {
          if (jj < i) continue;
          double q = 0.0;
#pragma unroll
          for (int k = 0; k < N; ++k) q = fma(A[k], rec(TO + jj * N + k), q);
          Qs[TR::at(i, jj) * NB] = q;
        }
      }
    };
    if (right) side(std::true_type{});
    else side(std::false_type{});
  }
  __syncthreads();                   // Q_l, Q_r complete; T_l, T_r dead
  double *Stt = REC + col * NN;      // [32][NN] dense rows: the store box
  if (active) {
    const double *Q0 = SNB + col;
#pragma unroll
    for (int i = 0; i < N; ++i)
#pragma unroll
      for (int jj = i; jj < N; ++jj) {
        const int e = TR::at(i, jj);
        if ((e * 2) / NT == (right ? 1 : 0)) {
          const double sv = (rec(RR::P + e) - Q0[e * NB]) - Q0[(NT + e) * NB];
          Stt[i * N + jj] = sv;
          Stt[jj * N + i] = sv;
        }
      }
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (tid == 0) {
    tma_store2d(&m.Sout, 0, (int)b0, REC);
    if (a.do_state) tma_store2d(&m.xout, 0, (int)b0, XST);
    if (KS_BWD_XSTAGE && a.Xcur.p) {   // the tile's two cross-array tiles (fewer at the level end)
      const int64_t xt = 2 * (int64_t)blockIdx.x, xtiles = (a.K + 1 + BC - 1) / BC;
      const int nt = xtiles - xt >= 2 ? 2 : (int)(xtiles - xt);
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(a.Xcur.p + xt * a.Xcur.ts),
                   "r"(smem_u32(bsm + L::XCS)), "r"((unsigned)(nt * NN * BC * 8))
                   : "memory");
    }
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
  }
}

// Host: the four tensor maps of one level (cuTensorMapEncodeTiled through the
// runtime's driver entry point: no libcuda link dependency).
static PFN_cuTensorMapEncodeTiled_v12000 tmap_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 f = nullptr;
  if (!f) {
    cudaDriverEntryPointQueryResult q;
    void *p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      f = (PFN_cuTensorMapEncodeTiled_v12000)p;
  }
  return f;
}
static bool tmap_rows(CUtensorMap *m, const double *base, int width, int64_t rows, int64_t pitch, int box) {
  auto enc = tmap_encoder();
  if (!enc || rows < 1 || rows > INT32_MAX) return false;
  const cuuint64_t dims[2] = {(cuuint64_t)width, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)(pitch * 8)};
  const cuuint32_t boxd[2] = {(cuuint32_t)width, (cuuint32_t)box};
  const cuuint32_t es[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, (void *)base, dims, strides, boxd, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
             CU_TENSOR_MAP_SWIZZLE_NONE, (CUtensorMapL2promotion)KS_TMAP_PROMO,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
// true: launched (even n, a regular level with at least one neighbour column)
template <int N>
bool backward_tma(const SmallBackwardArgs &a, cudaStream_t s) {
  if constexpr (N % 2 != 0) {
    return false;
  } else {
    const int64_t nc = (a.K + 1) / 2, Kup = a.K / 2, st = 2ll << a.shift;
    if (!KS_BWD_TMA || !a.do_cov || Kup < 1) return false;
    BwdMaps m;
    const double *xb = a.x ? a.x : a.S;   // do_state == 0: never dereferenced
    if (!tmap_rows(&m.Sout, a.S + ((1ll << a.shift) - 1) * N * N, N * N, nc, st * N * N, kBwdCols) ||
        !tmap_rows(&m.Snb, a.S + (st - 1) * N * N, N * N, Kup, st * N * N, kBwdCols + 1) ||
        !tmap_rows(&m.xout, xb + ((1ll << a.shift) - 1) * N, N, nc, st * N, kBwdCols) ||
        !tmap_rows(&m.xnb, xb + (st - 1) * N, N, Kup, st * N, kBwdCols + 1))
      return false;
    const bool xst = KS_BWD_XSTAGE && a.Xcur.p;
    const size_t smem = (xst ? BwdT<N>::total_x : BwdT<N>::total) * sizeof(double);
    set_smem_attr((const void *)small_backward_tma_kernel<N>, (int)(BwdT<N>::total_x * sizeof(double)));
    small_backward_tma_kernel<N><<<(unsigned)((nc + kBwdCols - 1) / kBwdCols), 2 * kBwdCols, smem, s>>>(a, m);
    return true;
  }
}

// ---------------------------------------------------------------- whiten ---

// Store element e of column i of a whitened level-0 view (constant: ES = 1).
__device__ __forceinline__ void wst(const TView &v, int cst, int64_t i, int e, double x) {
  if (cst) stv<1>(v, i, e, x);
  else stv<64>(v, i, e, x);
}

// Exponent range of the Givens path (the empty-row prior d = 2^-600, see
// kEmptyRow): a whitened block column with squared norm outside
// [1e-160, 1e120] (norm outside [1e-80, 1e60]) could be biased by the prior
// (relative 2^-600 / |y|^2 > 1e-21) or overflow y_k^2 rho (|y| > 6.6e63);
// such a problem is rejected (KS_ERR_ARG from ks_sync_status) instead of
// being solved inaccurately.  Zero blocks (no rows) are fine.
__device__ __forceinline__ bool out_of_range(double sq) { return sq != 0.0 && !(sq >= 1e-160 && sq <= 1e120); }

// Evolution blocks: K = Lam Lam^T (Cholesky), El = -Lam^{-1}F,
// Er = Lam^{-1}, e = Lam^{-1} c.  One thread per distinct block.
template <int N, bool PRE = false>
__device__ __forceinline__ void whiten_evo_body(const SmallWhitenArgs &a, int64_t i) {
  if (i >= a.cntE) return;
  const int64_t g = a.first_global + i;
  // no evolution row: the first step of the (global) problem, and of every
  // problem of a batch (step g with g % seg == 0)
  const bool evo = !((a.cntE != 1 && g % a.seg == 0) || (a.N == 1 && a.first_global == 0));
  if (!evo) {
#pragma unroll
    for (int k = 0; k < N * N; ++k) {
      wst(a.El, a.cE, i, k, 0.0);
      wst(a.Er, a.cE, i, k, 0.0);
    }
#pragma unroll
    for (int k = 0; k < N; ++k) wst(a.e, a.cE, i, k, 0.0);
    wst(a.nEr, a.cE, i, 0, 0.0);
    wst(a.nEl, a.cE, i, 0, 0.0);
    return;
  }
  const int64_t iK = (a.cntE == 1) ? 0 : i;
  const double *K = a.K + iK * a.sK, *F = a.F + iK * a.sF;
  const double *cc = a.c ? a.c + iK * a.sc : nullptr;
  // general model: l_i evolution rows, H_i (l_i x n_i), F_i
  // (l_i x n_{i-1}); the unused rows / columns of the uniform n x n blocks are
  // masked to zero (K: identity), so rows >= l_i of El, Er, e come out zero
  const int li = a.l ? a.l[i] : (a.ns ? a.ns[i] : N);
  const int ni = a.ns ? a.ns[i] : N;
  const int npv = (a.ns && i > 0) ? a.ns[i - 1] : N;
  const double *Hv = a.Hev ? a.Hev + iK * a.sHev : nullptr;
  double Lm[N][N];
  bool ok = true;
#pragma unroll
  for (int r = 0; r < N; ++r)
#pragma unroll
    for (int c = 0; c <= r; ++c) Lm[r][c] = (r < li) ? K[r * N + c] : (r == c ? 1.0 : 0.0);
  if (a.chol) {   // KS_COV_IS_CHOL: K holds Lam itself (nonzero diagonal)
#pragma unroll
    for (int j = 0; j < N; ++j) {
      const bool g = Lm[j][j] != 0.0 && Lm[j][j] - Lm[j][j] == 0.0;
      ok &= g;
      if (!g) Lm[j][j] = 1.0;   // continue with a finite factor (outputs undefined, status recorded)
    }
  } else {
#pragma unroll
    for (int j = 0; j < N; ++j) {
      double d = Lm[j][j];
#pragma unroll
      for (int k = 0; k < j; ++k) d = fma(-Lm[j][k], Lm[j][k], d);
      ok &= d > 0.0;
      const double ljj = sqrt(d > 0.0 ? d : 1.0), il = 1.0 / ljj;
      Lm[j][j] = ljj;
#pragma unroll
      for (int r = j + 1; r < N; ++r) {
        double v = Lm[r][j];
#pragma unroll
        for (int k = 0; k < j; ++k) v = fma(-Lm[r][k], Lm[j][k], v);
        Lm[r][j] = v * il;
      }
    }
  }
  if (!ok) report(a.status, (a.cntE == 1) ? (a.first_global == 0 ? 1 : 0) : i, kBadK);
  double il[N];
#pragma unroll
  for (int r = 0; r < N; ++r) il[r] = 1.0 / Lm[r][r];
  double nel = 0.0, ner = 0.0;
  // PRE (the one-thread launch of a constant model, pure latency): F and c
  // are read before any output is stored -- the stores below may alias them
  // for the compiler, which then issues each column's loads only after the
  // previous column's stores (a DRAM round trip per column).  Per-step
  // launches keep the loads in the loop (the preload's registers cost
  // occupancy there: c3 whitening 50 -> 66 us).
  double Fv[N][N], cv[N];
  if (PRE) {
#pragma unroll
    for (int r = 0; r < N; ++r) {
#pragma unroll
      for (int c = 0; c < N; ++c) Fv[r][c] = (r < li && c < npv) ? __ldg(F + r * N + c) : 0.0;
      cv[r] = (cc && r < li) ? __ldg(cc + r) : 0.0;
    }
  }
  // El = -Lam^{-1} F, column by column
#pragma unroll
  for (int c = 0; c < N; ++c) {
    double x[N];
#pragma unroll
    for (int r = 0; r < N; ++r) {
      double s = PRE ? Fv[r][c] : ((r < li && c < npv) ? F[r * N + c] : 0.0);
#pragma unroll
      for (int k = 0; k < r; ++k) s = fma(-Lm[r][k], x[k], s);
      x[r] = s * il[r];
    }
#pragma unroll
    for (int r = 0; r < N; ++r) {
      wst(a.El, a.cE, i, r * N + c, -x[r]);
      nel = fma(x[r], x[r], nel);
    }
  }
  // Er = Lam^{-1} H_i (H_i = I: lower triangular Lam^{-1})
#pragma unroll
  for (int c = 0; c < N; ++c) {
    double x[N];
#pragma unroll
    for (int r = 0; r < N; ++r) {
      double s = (r < li && c < ni) ? (Hv ? __ldg(Hv + r * N + c) : (r == c ? 1.0 : 0.0)) : 0.0;
#pragma unroll
      for (int k = 0; k < r; ++k) s = fma(-Lm[r][k], x[k], s);
      x[r] = s * il[r];
    }
#pragma unroll
    for (int r = 0; r < N; ++r) {
      wst(a.Er, a.cE, i, r * N + c, x[r]);
      ner = fma(x[r], x[r], ner);
    }
  }
  {
    double x[N];
#pragma unroll
    for (int r = 0; r < N; ++r) {
      double s = PRE ? cv[r] : ((cc && r < li) ? cc[r] : 0.0);
#pragma unroll
      for (int k = 0; k < r; ++k) s = fma(-Lm[r][k], x[k], s);
      x[r] = s * il[r];
      wst(a.e, a.cE, i, r, x[r]);
    }
  }
  wst(a.nEr, a.cE, i, 0, ner);
  wst(a.nEl, a.cE, i, 0, nel);
  if (out_of_range(ner) || out_of_range(nel))
    report(a.status, (a.cntE == 1) ? (a.first_global == 0 ? 1 : 0) : i, kBadScale);
}

// Observation blocks: L = M M^T; C = M^{-1} H, y = M^{-1} o (rows >= m_i are 0).
// One thread per distinct block; m_i <= kSmallMaxM.
template <int N, bool PRE = false>
__device__ __forceinline__ void whiten_obs_body(const SmallWhitenArgs &a, int64_t i) {
  constexpr int MM = kSmallMaxM;
  if (i >= a.cntC) return;
  const int mx = a.m_max;
  const int mi = a.m ? a.m[i] : mx;
  const double *L = a.L + i * a.sL, *H = a.H + i * a.sH, *o = a.o + i * a.so;
  const int ni = a.ns ? a.ns[i] : N;   // general model: columns >= n_i of H_i ignored
  double Lm[MM][MM];
  bool ok = true;
  if (a.chol) {   // KS_COV_IS_CHOL: L holds M itself (nonzero diagonal)
#pragma unroll
    for (int r = 0; r < MM; ++r)
#pragma unroll
      for (int k = 0; k <= r; ++k)
        if (r < mi) {
          Lm[r][k] = L[r * mx + k];
          if (k == r) {
            const bool g = Lm[r][r] != 0.0 && Lm[r][r] - Lm[r][r] == 0.0;
            ok &= g;
            if (!g) Lm[r][r] = 1.0;
          }
        }
  } else {
#pragma unroll
    for (int j = 0; j < MM; ++j) {
      if (j < mi) {
        double d = L[j * mx + j];
#pragma unroll
        for (int k = 0; k < j; ++k) d = fma(-Lm[j][k], Lm[j][k], d);
        ok &= d > 0.0;
        const double ljj = sqrt(d > 0.0 ? d : 1.0), il = 1.0 / ljj;
        Lm[j][j] = ljj;
#pragma unroll
        for (int r = j + 1; r < MM; ++r) {
          if (r < mi) {
            double v = L[r * mx + j];
#pragma unroll
            for (int k = 0; k < j; ++k) v = fma(-Lm[r][k], Lm[j][k], v);
            Lm[r][j] = v * il;
          }
        }
      }
    }
  }
  if (!ok) report(a.status, i, kBadL);
  if (a.Mall) {   // KS_KEEP_WHITENING: M_i for ks_update_obs
#pragma unroll
    for (int r = 0; r < MM; ++r)
#pragma unroll
      for (int k = 0; k < MM; ++k)
        if (r < mx && k < mx) a.Mall[i * (int64_t)mx * mx + r * mx + k] = (k <= r && r < mi) ? Lm[r][k] : 0.0;
  }
  double ild[MM];   // reciprocal diagonal (multiplications in the solves below)
#pragma unroll
  for (int r = 0; r < MM; ++r) ild[r] = (r < mi) ? 1.0 / Lm[r][r] : 0.0;
  double nc = 0.0;
  // PRE: H and o read before any output is stored (see whiten_evo_body)
  double Hr[MM][N + 1];
  if (PRE) {
#pragma unroll
    for (int r = 0; r < MM; ++r) {
#pragma unroll
      for (int c = 0; c < N; ++c) Hr[r][c] = (r < mi && c < ni) ? __ldg(H + r * N + c) : 0.0;
      Hr[r][N] = (r < mi && !a.constC) ? __ldg(o + r) : 0.0;
    }
  }
#pragma unroll
  for (int c = 0; c <= N; ++c) {          // N columns of H, then o
    const bool is_o = (c == N);
    if (is_o && a.constC) break;
    double x[MM];
#pragma unroll
    for (int r = 0; r < MM; ++r) {
      if (r < mi) {
        double s = PRE ? Hr[r][c] : (is_o ? o[r] : (c < ni ? H[r * N + c] : 0.0));
#pragma unroll
        for (int k = 0; k < r; ++k) s = fma(-Lm[r][k], x[k], s);
        x[r] = s * ild[r];
      } else {
        x[r] = 0.0;
      }
    }
#pragma unroll
    for (int r = 0; r < MM; ++r) {
      if (r < a.RC) {
        if (is_o) {
          wst(a.y, 0, i, r, x[r]);
        } else {
          // rows m_i .. m_i + n - n_i - 1: the padding rows e_k^T x_i = 0
          // (k = n_i ..) of the general model's embedding (y = 0)
          const double v = (r < mi) ? x[r] : ((r - mi < N - ni && c == ni + (r - mi)) ? 1.0 : 0.0);
          wst(a.C, a.cC, i, r * N + c, v);
          nc = fma(v, v, nc);
        }
      }
    }
  }
  wst(a.nC, a.cC, i, 0, nc);
  if (out_of_range(nc)) report(a.status, i, kBadScale);
  if (a.constC) {
#pragma unroll
    for (int r = 0; r < MM; ++r)
#pragma unroll
      for (int k = 0; k < MM; ++k)
        if (r < mx && k < mx) a.Mchol[r * mx + k] = (k <= r && r < mi) ? Lm[r][k] : 0.0;
    if (a.Minv) {   // M^{-1} (lower triangular) for the factor's fused y = M^{-1} o
#pragma unroll
      for (int c = 0; c < MM; ++c) {
        double x[MM];
#pragma unroll
        for (int r = 0; r < MM; ++r) {
          double sv = (r == c) ? 1.0 : 0.0;
#pragma unroll
          for (int k = 0; k < r; ++k) sv = fma(-Lm[r][k], x[k], sv);
          x[r] = (r < mi && r >= c) ? sv * ild[r] : 0.0;
        }
#pragma unroll
        for (int r = 0; r < MM; ++r)
          if (r < mx && c < mx) a.Minv[r * mx + c] = x[r];
      }
    }
  }
}

// Evolution and observation blocks in one launch (independent): CTAs
// [0, gE) whiten the evolution blocks, the rest the observation blocks.
// The two halves as separate kernels (each body alone in the instruction cache)
template <int N, bool PRE = false>
__global__ void __launch_bounds__(128) small_whiten_e(SmallWhitenArgs a) {
  whiten_evo_body<N, PRE>(a, (int64_t)blockIdx.x * blockDim.x + threadIdx.x);
}
template <int N, bool PRE = false>
__global__ void __launch_bounds__(128) small_whiten_o(SmallWhitenArgs a) {
  whiten_obs_body<N, PRE>(a, (int64_t)blockIdx.x * blockDim.x + threadIdx.x);
}

// Constant observation model: y_i = M^{-1} o_i, one thread per step.
template <int DUMMY>
__global__ void __launch_bounds__(256) small_whiten_y(SmallWhitenArgs a) {
  __shared__ double M[kSmallMaxM * kSmallMaxM], Mi[kSmallMaxM];
  const int mx = a.m_max;
  for (int k = threadIdx.x; k < mx * mx; k += blockDim.x) M[k] = a.Mchol[k];
  for (int k = threadIdx.x; k < mx; k += blockDim.x) Mi[k] = 1.0 / a.Mchol[k * mx + k];
  __syncthreads();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.N) return;
  const double *o = a.o + i * a.so;
  double y[kSmallMaxM];
#pragma unroll
  for (int r = 0; r < kSmallMaxM; ++r) {
    if (r < mx) {
      double s = o[r];
#pragma unroll
      for (int k = 0; k < r; ++k) s = fma(-M[r * mx + k], y[k], s);
      y[r] = s * Mi[r];
      wst(a.y, 0, i, r, y[r]);
    }
  }
}

template <int N, bool L0, bool CE, bool CC, bool OAOS, bool ZS = false>
cudaError_t factor_launch(const SmallFactorArgs &a, cudaStream_t s) {
  const int T = 64;
  const int64_t np = (a.K >= 2 ? a.K / 2 : 1) + (ZS ? 1 : 0);
  const unsigned g = (unsigned)((np + T - 1) / T);
  const size_t smem = ((size_t)T * kParkDoubles<N> + CstOff<N>::size) * sizeof(double);
  set_smem_attr((const void *)small_factor_kernel<N, L0, CE, CC, OAOS, ZS>, (int)smem);
  small_factor_kernel<N, L0, CE, CC, OAOS, ZS><<<g, T, smem, s>>>(a);
  return cudaGetLastError();
}

template <int N, bool OAOS>
cudaError_t factor_oaos(const SmallFactorArgs &a, cudaStream_t s) {
  const int64_t npairs = a.K >= 2 ? a.K / 2 : 1;
  int dev = 0, sms = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (a.in.ent.p != nullptr && npairs <= (int64_t)64 * sms && !std::getenv("KS_NO_SPLIT_LEVELS")) {
    // latency-bound level (one 64-pair CTA per SM at most): three threads per pair
    const size_t smem = ((size_t)64 * kParkSP<N> + CstOff<N>::size) * sizeof(double);
    set_smem_attr((const void *)small_factor_split_kernel<N, OAOS>, (int)smem);
    small_factor_split_kernel<N, OAOS><<<(unsigned)((npairs + 63) / 64), kTailThreads, smem, s>>>(a);
    return cudaGetLastError();
  }
  if (a.in.ent.p != nullptr)   // level >= 1; an odd level splits its last column off (split_odd)
    return split_odd(a.K, 64) ? factor_launch<N, false, false, false, OAOS, true>(a, s)
                              : factor_launch<N, false, false, false, OAOS>(a, s);
  if (a.cE) {
    if (a.cC) return factor_launch<N, true, true, true, OAOS>(a, s);
    return factor_launch<N, true, true, false, OAOS>(a, s);
  }
  if (a.cC) return factor_launch<N, true, false, true, OAOS>(a, s);
  return factor_launch<N, true, false, false, OAOS>(a, s);
}

template <int N>
cudaError_t factor_n(const SmallFactorArgs &a, cudaStream_t s) {
  return a.outAoS ? factor_oaos<N, true>(a, s) : factor_oaos<N, false>(a, s);
}

template <int N>
cudaError_t factor_tail_n(const SmallTailArgs &t, cudaStream_t s) {
  const size_t smem = tail_smem_bytes<N>();
  set_smem_attr((const void *)small_factor_tail_kernel<N>, (int)smem);
  small_factor_tail_kernel<N><<<(unsigned)(t.W ? t.K[0] / t.W : 1), kTailThreads, smem, s>>>(t);
  return cudaGetLastError();
}
template <int N>
int tail_cols_n() { return tail_max_cols<N>(); }

template <int N>
cudaError_t backward_n(const SmallBackwardArgs &a, cudaStream_t s) {
  if (backward_tma<N>(a, s)) return cudaGetLastError();
  const int64_t nc = (a.K + 1) / 2;
  const size_t full = bwd_smem_doubles<N>() * sizeof(double);
  const size_t smem = a.do_cov ? full : 0;
  set_smem_attr((const void *)small_backward_kernel<N>, (int)full);
  small_backward_kernel<N><<<(unsigned)((nc + kBwdCols - 1) / kBwdCols), 2 * kBwdCols, smem, s>>>(a);
  return cudaGetLastError();
}

template <int N>
cudaError_t backward_tail_n(const SmallBwdTailArgs &t, cudaStream_t s) {
  const size_t smem = 2 * bwd_smem_doubles<N>() * sizeof(double);
  set_smem_attr((const void *)small_backward_tail_kernel<N>, (int)smem);
  small_backward_tail_kernel<N><<<(unsigned)(t.W ? t.nsub : 1), 4 * kBwdCols, smem, s>>>(t);
  return cudaGetLastError();
}

template <int N>
cudaError_t whiten_n(const SmallWhitenArgs &a, cudaStream_t s, int *nl) {
  const int T = 128;
  const unsigned gE = (unsigned)((a.cntE + T - 1) / T);
  const unsigned gC = a.RC > 0 ? (unsigned)((a.cntC + T - 1) / T) : 0u;
  // two launches, each body alone in the instruction cache (one combined
  // kernel branching on blockIdx measured 27 % no-instruction stalls; c3
  // whitening 58 -> 50 us, c2 86 -> 83 us)
  // (one distinct block: the latency-bound one-thread launch preloads its inputs)
  if (a.cntE == 1) small_whiten_e<N, true><<<gE, T, 0, s>>>(a);
  else small_whiten_e<N><<<gE, T, 0, s>>>(a);
  *nl = 1;
  if (gC) {
    if (a.cntC == 1) small_whiten_o<N, true><<<gC, T, 0, s>>>(a);
    else small_whiten_o<N><<<gC, T, 0, s>>>(a);
    *nl += 1;
  }
  if (a.m_max > 0) {
    if (a.constC && !a.Minv) {   // (with Minv the factor computes y = M^{-1} o itself)
      small_whiten_y<N><<<(unsigned)((a.N + 255) / 256), 256, 0, s>>>(a);
      *nl += 1;
    }
  }
  return cudaGetLastError();
}

}  // namespace smalld
}  // namespace ks

