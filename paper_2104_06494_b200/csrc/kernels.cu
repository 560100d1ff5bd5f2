// Region-store kernels (see kernels.cuh).  All are HBM/latency bound; the
// data layout is axis-major SoA (low[a*cap + j]) so every per-region access
// is coalesced across the warp, and children of kept region k are written
// as 16-byte pairs (2k, 2k+1).
#include "kernels.cuh"

#include <algorithm>
#include <cstdlib>
#include <mutex>
#include <set>
#include <utility>
#include <limits>

#include "glibc_tables.h"

namespace pgn {

namespace {

__device__ const uint64_t g_exp_tab[256] = PGN_EXP_TAB_INIT;
__device__ const uint64_t g_sincos_tab[440] = PGN_SINCOS_TAB_INIT;

inline unsigned grid_for(int64_t work, int threads) {
  return static_cast<unsigned>((work + threads - 1) / threads);
}

// ---- uniform split ----------------------------------------------------------
__global__ void k_uniform_split(int n, int d, int64_t m, int64_t cap, double* low, double* len,
                                const double* lower, const double* step, int64_t first) {
  const int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= m) return;
  int64_t rem = first + j;  // global region index
  for (int a = 0; a < n; ++a) {  // geometry.cpp:100-110, axis 0 fastest
    const int64_t cell = rem % d;
    rem /= d;
    low[a * cap + j] = P_ADD(lower[a], P_MUL(static_cast<double>(cell), step[a]));
    len[a * cap + j] = step[a];
  }
}

// ---- deterministic block folds ----------------------------------------------
// One thread per (block, quantity): the serial left fold over <= 2048 values
// (reduce.cpp:36-43 / 54-62).  The fold is a dependent DADD chain, so the
// loads are batched 8 ahead.  Masked folds add +0.0 for skipped entries,
// which equals skipping: the running sum starts at +0.0 and can never become
// -0.0 under round-to-nearest.
template <bool MASKED>
__device__ __forceinline__ double serial_fold(const double* __restrict__ x,
                                              const uint8_t* __restrict__ f, uint8_t which,
                                              int64_t lo, int64_t hi, int64_t* cnt_other) {
  double s = 0.0;
  int64_t c = 0;
  int64_t i = lo;
  for (; i + 8 <= hi; i += 8) {
    double v[8];
    uint8_t g[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      v[u] = __ldg(x + i + u);
      if (MASKED) g[u] = __ldg(f + i + u);
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      if (MASKED) {
        const bool take = g[u] == which;
        c += take ? 0 : 1;
        s = P_ADD(s, take ? v[u] : 0.0);
      } else {
        s = P_ADD(s, v[u]);
      }
    }
  }
  for (; i < hi; ++i) {
    const double v = __ldg(x + i);
    if (MASKED) {
      const bool take = __ldg(f + i) == which;
      c += take ? 0 : 1;
      s = P_ADD(s, take ? v : 0.0);
    } else {
      s = P_ADD(s, v);
    }
  }
  if (cnt_other) *cnt_other = c;
  return s;
}

// One CTA per 2048-block: the block is staged in shared memory with
// coalesced loads, then the strict serial folds run from smem (the chain is a
// dependent DADD sequence, so the only thing that matters is that each step
// waits on DADD latency, not on a global load).  The est chains and the err
// chains run on lane 0 of two different warps so they issue in parallel.
constexpr int kFoldThreads = 256;

struct FoldSmem {
  double est[kBlock];
  double err[kBlock];
  uint8_t flag[kBlock];
};

__device__ __forceinline__ int64_t stage_block(FoldSmem& S, const double* __restrict__ est,
                                               const double* __restrict__ err,
                                               const uint8_t* __restrict__ flag, int64_t lo,
                                               int cnt, bool need_est, double t, bool probe) {
  int active = 0;
  for (int i = threadIdx.x; i < kBlock; i += kFoldThreads) {
    bool a = false;
    if (i < cnt) {
      const double e = __ldg(err + lo + i);
      uint8_t f = __ldg(flag + lo + i);
      if (probe) f = (f && !(e < t)) ? 1 : 0;  // candidate (classify.cpp:63-66)
      S.err[i] = e;
      S.flag[i] = f;
      if (need_est) S.est[i] = __ldg(est + lo + i);
      a = f != 0;
    }
    active += __syncthreads_count(a);
  }
  return active;
}

// q0 = sum est, q1 = sum err, q2 = sum est[flag==0], q3 = sum err[flag==0],
// cnt = #flag==1   (reduce.cpp:31-64 via driver.cpp:145-146, classify.cpp:104-108)
__global__ void __launch_bounds__(kFoldThreads)
    k_fold_eval(int64_t m, int64_t nblk, const double* __restrict__ est,
                const double* __restrict__ err, const uint8_t* __restrict__ flag, double* part,
                int64_t* cnt, int use_t, double t) {
  __shared__ FoldSmem S;
  const int64_t b = blockIdx.x;
  const int64_t lo = b * kBlock;
  const int n = static_cast<int>(m - lo < kBlock ? m - lo : kBlock);
  // use_t: fold under the final flags of threshold t (classify.cpp:63-66)
  const int64_t active = stage_block(S, est, err, flag, lo, n, true, t, use_t != 0);
  if ((threadIdx.x & 31) != 0 || threadIdx.x >= 64) {
    if (threadIdx.x == 64) cnt[b] = active;
    return;
  }
  const double* x = threadIdx.x == 0 ? S.est : S.err;
  double all = 0.0, fin = 0.0;
#pragma unroll 8
  for (int i = 0; i < n; ++i) {
    const double v = x[i];
    all = P_ADD(all, v);
    fin = P_ADD(fin, S.flag[i] ? 0.0 : v);
  }
  const int q = threadIdx.x == 0 ? 0 : 1;
  part[q * nblk + b] = all;
  part[(q + 2) * nblk + b] = fin;
}

// Pairwise tree (reduce.cpp:13-27: p[i] = p[2i] + p[2i+1], odd tail carried)
// of src[0..n) by a group of gn threads (local id lt).  The first level reads
// the global partials, every later level runs in shared memory (`sm`, room for
// n + 64 doubles): one __syncthreads per level instead of an L2 round trip.
// Every thread of the CTA must call it with the same n (it syncs the CTA).
__device__ __forceinline__ double tree_sum_smem(const double* src, int64_t n, double* sm, int lt,
                                                int gn) {
  if (n <= 0) return 0.0;
  const double* s = src;
  double* d = sm;
  int64_t cur = n;
  if (cur > 1) {  // first level from global memory: a thread's loads all in flight at once
    constexpr int K = 8;
    const int64_t half = cur / 2;
    for (int64_t base = 0; base < half; base += static_cast<int64_t>(gn) * K) {
      double a[K], b[K];
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const int64_t i = base + lt + static_cast<int64_t>(k) * gn;
        a[k] = i < half ? s[2 * i] : 0.0;
        b[k] = i < half ? s[2 * i + 1] : 0.0;
      }
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const int64_t i = base + lt + static_cast<int64_t>(k) * gn;
        if (i < half) d[i] = P_ADD(a[k], b[k]);
      }
    }
    if ((cur & 1) && lt == 0) d[half] = s[cur - 1];
    __syncthreads();
    cur = half + (cur & 1);
    s = d;
    d += cur;
  }
  while (cur > 1) {
    const int64_t half = cur / 2;
    for (int64_t i = lt; i < half; i += gn) d[i] = P_ADD(s[2 * i], s[2 * i + 1]);
    if ((cur & 1) && lt == 0) d[half] = s[cur - 1];
    __syncthreads();
    cur = half + (cur & 1);
    s = d;
    d += cur;
  }
  return s[0];
}
// Shared-memory trees are used while they fit: doubles per tree = nblk + 64.
constexpr int64_t kTreeSmemMaxBytes = 200 * 1024;
inline size_t tree_smem_bytes(int64_t nblk, int groups) {
  return static_cast<size_t>(groups) * static_cast<size_t>(nblk + 64) * sizeof(double);
}

// Speculative threshold probes: T <= kMaxProbes candidate thresholds (a
// level-order tree of the search's possible next steps, classify.cpp:82-89)
// evaluated in ONE pass over the block.
//
// Per 2048-block the result is 2T strict serial folds (sum err / sum est over
// the non-candidates of each threshold, reduce.cpp:54-62) -- dependent DADD
// chains, so the kernel is built around keeping 30 chains busy on ONE warp:
// lane j < 15 folds err for node j, lane 16+j folds est for node j.  The
// candidate test is one predicate-producing LOP3: producers give every region
// a code (flag ? #{sorted thresholds the error reaches} : 0, see ProbeSet),
// stored as the 16-bit mask (1 << code) - 1 over sorted positions, and node
// j's candidates are exactly the regions with bit pos[j] set.  Each step is
// then LOP3 + 2 FSEL + DADD (+ 3/8 LDS.128); candidate counts come from a
// per-block code histogram the producers build with warp-aggregated atomics.
//
// Streaming: warps 1..3 stage chunk c+1 (est, err, code; 17 B/region) into a
// 2-deep shared-memory ring while warp 0 folds chunk c, so a CTA needs only
// 13.9 KB and every block of a 2^22-region batch is resident at once.
constexpr int kProbeThreads = 128;
#ifndef PGN_PROBE_UNROLL
#define PGN_PROBE_UNROLL 2
#endif
constexpr int kProbeUnroll = PGN_PROBE_UNROLL;
constexpr int kProbeChunk = 384;  // = 4 x 96 producer threads = 3 x 128
#ifndef PGN_PROBE_LDS_PIPE
#define PGN_PROBE_LDS_PIPE 1
#endif
#ifndef PGN_PROBE_PIPE
#define PGN_PROBE_PIPE 1  // producers keep the next chunk's loads in flight across a barrier
#endif
struct ProbeStage {
  double err[2][kProbeChunk];
  double est[2][kProbeChunk];
  uint16_t mask[2][kProbeChunk];
  double s[16];
  unsigned hist[17];  // regions per code (candidate counts = suffix sums)
};

// ss: the 16 sorted thresholds in shared memory (lane-divergent indices would
// serialise in the constant cache).
__device__ __forceinline__ uint8_t probe_code(const double* ss, int nan_cnt, uint8_t f, double e) {
  if (!f) return 0;
  if (e != e) return 16;
  int p = 0;  // upper bound over 16 sorted entries (NaN padding compares false)
#pragma unroll
  for (int step = 8; step > 0; step >>= 1)
    if (ss[p + step - 1] <= e) p += step;
  return static_cast<uint8_t>(nan_cnt + p);
}

// Stage chunk c (kProbeChunk regions) into ring slot c & 1: nt threads, PER
// regions each (nt * PER == kProbeChunk).  Split in two halves so the
// producers can software-pipeline: probe_load issues the chunk's global loads
// into registers, probe_store (one barrier interval later) turns them into
// codes + ring entries -- the loads of chunk c + 2 are in flight while the
// folding warp works through chunk c.
template <int PER>
struct ProbeRegs {
  double e[PER], v[PER];
  uint8_t f[PER];
};
template <int PER>
__device__ __forceinline__ void probe_load(ProbeRegs<PER>& R, const double* __restrict__ est,
                                           const double* __restrict__ err,
                                           const uint8_t* __restrict__ flag, int64_t lo, int n,
                                           int c, int t0, int nt) {
#pragma unroll
  for (int u = 0; u < PER; ++u) {
    const int k = c * kProbeChunk + t0 + u * nt;
    R.e[u] = 0.0;
    R.v[u] = 0.0;
    R.f[u] = 0;
    if (k < n) {
      R.e[u] = __ldg(err + lo + k);
      R.v[u] = __ldg(est + lo + k);
      R.f[u] = __ldg(flag + lo + k);
    }
  }
}
template <int PER>
__device__ __forceinline__ void probe_store(ProbeStage& S, const ProbeSet& ts,
                                            const ProbeRegs<PER>& R, int c, int t0, int nt) {
  const int buf = c & 1;
#pragma unroll
  for (int u = 0; u < PER; ++u) {
    const int i = t0 + u * nt;
    const uint8_t code = probe_code(S.s, ts.nan_cnt, R.f[u], R.e[u]);
    // one shared atomic per distinct code in the warp (padding regions past
    // the block end have code 0, which no count reads)
    const unsigned peers = __match_any_sync(0xffffffffu, static_cast<unsigned>(code));
    if ((threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(&S.hist[code], __popc(peers));
    S.err[buf][i] = R.e[u];
    S.est[buf][i] = R.v[u];
    S.mask[buf][i] = static_cast<uint16_t>((1u << code) - 1u);
  }
}
template <int PER>
__device__ __forceinline__ void probe_stage_chunk(ProbeStage& S, const ProbeSet& ts,
                                                  const double* __restrict__ est,
                                                  const double* __restrict__ err,
                                                  const uint8_t* __restrict__ flag, int64_t lo,
                                                  int n, int c, int t0, int nt) {
  ProbeRegs<PER> R;
  probe_load<PER>(R, est, err, flag, lo, n, c, t0, nt);
  probe_store<PER>(S, ts, R, c, t0, nt);
}

// s += v unless (word & bit): the skip of reduce.cpp:59-60 as a predicated
// DADD (LOP3 -> predicate, @!P DADD: two instructions per step; the former
// select form, adding +0.0 for a skipped region, cost LOP3 + 2 FSEL + DADD).
#ifndef PGN_PROBE_PRED
#define PGN_PROBE_PRED 0  // measured slower on B200: ptxas if-converts it to DADD + 2 FSEL after the add, on the chain
#endif
__device__ __forceinline__ void add_unless(double& s, double v, uint32_t word, uint32_t bit) {
#if PGN_PROBE_PRED
  asm("{\n\t.reg .pred p;\n\tsetp.eq.b32 p, %2, 0;\n\t@p add.rn.f64 %0, %0, %1;\n\t}"
      : "+d"(s)
      : "d"(v), "r"(word & bit));
#else
  s = P_ADD(s, (word & bit) ? 0.0 : v);
#endif
}

__global__ void __launch_bounds__(kProbeThreads)
    k_probe_multi(int64_t m, int64_t nblk, const ProbeSet ts_arg, const double* __restrict__ est,
                  const double* __restrict__ err, const uint8_t* __restrict__ flag, double* part,
                  int64_t* cnt, const ProbeSet* dts) {
  __shared__ __align__(16) ProbeStage S;
  // dts: the speculative first pass, its ProbeSet built by k_finalize (the
  // predecessor of this programmatic launch)
  pdl_wait();
  const ProbeSet& ts = dts ? *dts : ts_arg;
  const int64_t b = blockIdx.x;
  const int64_t lo = b * kBlock;
  const int n = static_cast<int>(m - lo < kBlock ? m - lo : kBlock);
  const int nch = (n + kProbeChunk - 1) / kProbeChunk;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  if (tid < 16) S.s[tid] = ts.s[tid];
  if (tid < 17) S.hist[tid] = 0;
  __syncthreads();
  probe_stage_chunk<kProbeChunk / kProbeThreads>(S, ts, est, err, flag, lo, n, 0, tid,
                                                 kProbeThreads);
  __syncthreads();
  const int node = (lane & 15) < ts.T ? (lane & 15) : 0;
  const int pos = ts.pos[node];
  const int q = lane >> 4;  // 0: err chain, 1: est chain
  double fin = 0.0;
  constexpr int kPer = kProbeChunk / (kProbeThreads - 32);
  ProbeRegs<kPer> R;  // producers: chunk c + 1's loads, stored one interval later
  if (w > 0 && nch > 1) probe_load<kPer>(R, est, err, flag, lo, n, 1, tid - 32, kProbeThreads - 32);
  for (int c = 0; c < nch; ++c) {
    if (w > 0) {
      if (c + 1 < nch) {
#if PGN_PROBE_PIPE
        probe_store<kPer>(S, ts, R, c + 1, tid - 32, kProbeThreads - 32);
        if (c + 2 < nch) probe_load<kPer>(R, est, err, flag, lo, n, c + 2, tid - 32, kProbeThreads - 32);
#else
        probe_stage_chunk<kPer>(S, ts, est, err, flag, lo, n, c + 1, tid - 32, kProbeThreads - 32);
#endif
      }
    } else {
      const int buf = c & 1;
      const double* x = q ? S.est[buf] : S.err[buf];
      const uint16_t* mk = S.mask[buf];
      const int cntc = n - c * kProbeChunk < kProbeChunk ? n - c * kProbeChunk : kProbeChunk;
      if (cntc == kProbeChunk) {
        const uint32_t blo = 1u << pos, bhi = blo << 16;
#if PGN_PROBE_LDS_PIPE
        // register double buffer: group g + 1's shared-memory loads are issued
        // before group g's 8 dependent DADDs, so with one or two folding warps
        // per SM sub-partition the LDS latency is off the chain
        uint4 m8 = *reinterpret_cast<const uint4*>(mk);
        double2 v0 = *reinterpret_cast<const double2*>(x);
        double2 v1 = *reinterpret_cast<const double2*>(x + 2);
        double2 v2 = *reinterpret_cast<const double2*>(x + 4);
        double2 v3 = *reinterpret_cast<const double2*>(x + 6);
#pragma unroll 2
        for (int i = 0; i < kProbeChunk; i += 8) {
          const int nx = i + 8 < kProbeChunk ? i + 8 : i;  // last group: harmless reload
          const uint4 n8 = *reinterpret_cast<const uint4*>(mk + nx);
          const double2 n0 = *reinterpret_cast<const double2*>(x + nx);
          const double2 n1 = *reinterpret_cast<const double2*>(x + nx + 2);
          const double2 n2 = *reinterpret_cast<const double2*>(x + nx + 4);
          const double2 n3 = *reinterpret_cast<const double2*>(x + nx + 6);
          add_unless(fin, v0.x, m8.x, blo);
          add_unless(fin, v0.y, m8.x, bhi);
          add_unless(fin, v1.x, m8.y, blo);
          add_unless(fin, v1.y, m8.y, bhi);
          add_unless(fin, v2.x, m8.z, blo);
          add_unless(fin, v2.y, m8.z, bhi);
          add_unless(fin, v3.x, m8.w, blo);
          add_unless(fin, v3.y, m8.w, bhi);
          m8 = n8;
          v0 = n0;
          v1 = n1;
          v2 = n2;
          v3 = n3;
        }
#else
#pragma unroll kProbeUnroll
        for (int i = 0; i < kProbeChunk; i += 8) {
          const uint4 m8 = *reinterpret_cast<const uint4*>(mk + i);
          const double2 v0 = *reinterpret_cast<const double2*>(x + i);
          const double2 v1 = *reinterpret_cast<const double2*>(x + i + 2);
          const double2 v2 = *reinterpret_cast<const double2*>(x + i + 4);
          const double2 v3 = *reinterpret_cast<const double2*>(x + i + 6);
          add_unless(fin, v0.x, m8.x, blo);
          add_unless(fin, v0.y, m8.x, bhi);
          add_unless(fin, v1.x, m8.y, blo);
          add_unless(fin, v1.y, m8.y, bhi);
          add_unless(fin, v2.x, m8.z, blo);
          add_unless(fin, v2.y, m8.z, bhi);
          add_unless(fin, v3.x, m8.w, blo);
          add_unless(fin, v3.y, m8.w, bhi);
        }
#endif
      } else {
        for (int i = 0; i < cntc; ++i) add_unless(fin, x[i], mk[i], 1u << pos);
      }
    }
    __syncthreads();
  }
  if (w == 0 && (lane & 15) < ts.T) {
    part[(q * kMaxProbes + node) * nblk + b] = fin;
    if (q == 0) {
      int64_t c = 0;  // candidates of node j: regions whose code exceeds pos[j]
      for (int k = pos + 1; k <= 16; ++k) c += S.hist[k];
      cnt[node * nblk + b] = c;
    }
  }
}

// ---- fast probe pass -----------------------------------------------------------
// The threshold search's decisions need, per speculative threshold, the exact
// candidate count and the discarded error compared against a budget; only
// the ACCEPTED threshold's sums must be the reference's bits.  So a pass
// streams flag + err once (9 B/region, HBM-bound) and produces exact counts
// and fast sums in any order -- per thread, warp shuffles, one finalize CTA.
// The host treats a comparison as decided when |fast - budget| exceeds the
// sums' rounding bound (both orders are within gamma_2400 of the true sum of
// the nonnegative errors), falls back to the exact pass otherwise, and folds
// the accepted threshold exactly (k_fold_eval under the threshold).
constexpr int kPfThreads = 256;

__global__ void __launch_bounds__(kPfThreads)
    k_probe_fast(int64_t m, const ProbeSet ts, const double* __restrict__ err,
                 const uint8_t* __restrict__ flag, double* part, int64_t* cnt) {
  constexpr int W = kPfThreads / 32;
  __shared__ double s_s[16];
  __shared__ double s_acc[W][kMaxProbes];
  __shared__ long long s_c[W][kMaxProbes];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  if (tid < 16) s_s[tid] = ts.s[tid];
  __syncthreads();
  double acc[kMaxProbes];
  int c[kMaxProbes];
#pragma unroll
  for (int k = 0; k < kMaxProbes; ++k) {
    acc[k] = 0.0;
    c[k] = 0;
  }
  const int64_t stride = static_cast<int64_t>(gridDim.x) * kPfThreads;
#pragma unroll 4
  for (int64_t j = static_cast<int64_t>(blockIdx.x) * kPfThreads + tid; j < m; j += stride) {
    const double e = __ldg(err + j);
    const uint8_t code = probe_code(s_s, ts.nan_cnt, __ldg(flag + j), e);
#pragma unroll
    for (int k = 0; k < kMaxProbes; ++k) {
      const bool cand = code > ts.pos[k];
      acc[k] += cand ? 0.0 : e;
      c[k] += cand;
    }
  }
#pragma unroll
  for (int k = 0; k < kMaxProbes; ++k) {
    double a = acc[k];
    int cc = c[k];
    for (int o = 16; o > 0; o >>= 1) {
      a += __shfl_xor_sync(0xffffffffu, a, o);
      cc += __shfl_xor_sync(0xffffffffu, cc, o);
    }
    if (lane == 0) {
      s_acc[w][k] = a;
      s_c[w][k] = cc;
    }
  }
  __syncthreads();
  if (tid < kMaxProbes) {
    double a = 0.0;
    long long cc = 0;
#pragma unroll
    for (int q = 0; q < W; ++q) {
      a += s_acc[q][tid];
      cc += s_c[q][tid];
    }
    part[tid * gridDim.x + blockIdx.x] = a;
    cnt[tid * gridDim.x + blockIdx.x] = cc;
  }
}

// The accepted threshold's exact sums (reduce.cpp:31-64 under the final flags
// flag && !(err < t)): per 2048-block the CTA stages the masked estimates and
// errors (0.0 for candidates: adding +0.0 is the reference's skip) into
// shared memory with all its threads, then one thread per quantity folds the
// block strictly in order from shared memory, eight loads ahead of the DADD
// chain.  part[q * nblk + b]: q = 0 est, 1 err; cnt[b] = candidates.
constexpr int kFtThreads = 256;
__global__ void __launch_bounds__(kFtThreads)
    k_fold_threshold(int64_t m, int64_t nblk, const double* __restrict__ est,
                     const double* __restrict__ err, const uint8_t* __restrict__ flag, double t,
                     double* part, int64_t* cnt) {
  __shared__ __align__(16) double s_v[2][kBlock];
  const int64_t b = blockIdx.x;
  const int64_t lo = b * kBlock;
  const int n = static_cast<int>(m - lo < kBlock ? m - lo : kBlock);
  __shared__ int s_kept[kFtThreads / 32];
  int kept = 0;
#pragma unroll
  for (int r = 0; r < kBlock / kFtThreads; ++r) {  // all loads issued before any use
    const int i = r * kFtThreads + threadIdx.x;
    double e = 0.0, x = 0.0;
    bool k = false;
    if (i < n) {
      const uint8_t f = __ldg(flag + lo + i);
      e = __ldg(err + lo + i);
      x = __ldg(est + lo + i);
      k = f && !(e < t);  // candidate: stays active (classify.cpp:63-66)
    }
    s_v[0][i] = k ? 0.0 : x;
    s_v[1][i] = k ? 0.0 : e;
    kept += k;
  }
  for (int o = 16; o > 0; o >>= 1) kept += __shfl_xor_sync(0xffffffffu, kept, o);
  if ((threadIdx.x & 31) == 0) s_kept[threadIdx.x >> 5] = kept;
  __syncthreads();
  if (threadIdx.x == 0) {
    kept = 0;
#pragma unroll
    for (int w = 0; w < kFtThreads / 32; ++w) kept += s_kept[w];
  }
  if (threadIdx.x != 0 && threadIdx.x != 32) return;
  const int q = threadIdx.x >> 5;
  const double* v = s_v[q];
  double s = 0.0;
  const int n8 = n & ~7;
  for (int i = 0; i < n8; i += 8) {
    const double2 a = *reinterpret_cast<const double2*>(v + i);
    const double2 c = *reinterpret_cast<const double2*>(v + i + 2);
    const double2 d = *reinterpret_cast<const double2*>(v + i + 4);
    const double2 f = *reinterpret_cast<const double2*>(v + i + 6);
    s = P_ADD(s, a.x);
    s = P_ADD(s, a.y);
    s = P_ADD(s, c.x);
    s = P_ADD(s, c.y);
    s = P_ADD(s, d.x);
    s = P_ADD(s, d.y);
    s = P_ADD(s, f.x);
    s = P_ADD(s, f.y);
  }
  for (int i = n8; i < n; ++i) s = P_ADD(s, v[i]);
  part[q * nblk + b] = s;
  if (q == 0) cnt[b] = kept;
}

// Totals over the G CTAs of k_probe_fast into mapped host memory (err_sum =
// the fast sums, count exact), then publish `seq`.
__global__ void __launch_bounds__(512)
    k_probe_fast_total(int G, const double* part, const int64_t* cnt, ProbeScalars* out,
                       unsigned* ready, unsigned seq) {
  const int k = threadIdx.x >> 5, lane = threadIdx.x & 31;  // 16 warps: one per node
  double a = 0.0;
  long long n = 0;
  if (k < kMaxProbes) {
#pragma unroll 8
    for (int g = lane; g < G; g += 32) {  // independent loads, issued ahead
      a += part[k * G + g];
      n += cnt[k * G + g];
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, o);
    n += __shfl_xor_sync(0xffffffffu, n, o);
  }
  if (k < kMaxProbes && lane == 0) {
    out->err_sum[k] = a;
    out->est_sum[k] = 0.0;
    out->count[k] = n;
    __threadfence_system();
  }
  __syncthreads();
  if (threadIdx.x == 0 && ready) {
    __threadfence_system();
    *reinterpret_cast<volatile unsigned*>(ready) = seq;
  }
}

// Pairwise trees (reduce.cpp:13-27) for 2T fold arrays + T count totals:
// one CTA per array.
template <bool SMEM>
__global__ void __launch_bounds__(256)
    k_finalize_multi(int64_t nblk, int T, const double* part, const int64_t* cnt, double* scratch,
                     ProbeScalars* out, unsigned* ready, unsigned seq, int* done) {
  const int id = blockIdx.x;  // 0..2T-1 folds, 2T..3T-1 counts
  const int tid = threadIdx.x;
  pdl_wait();  // k_probe_multi's block records (launch_pdl)
  // zero-copy hand-off: `out` is mapped host memory; the last CTA to finish
  // publishes `seq` once every CTA's field is fenced (no D2H copy + sync)
  auto publish = [&] {
    if (!ready || tid != 0) return;
    __threadfence_system();
    if (atomicAdd(done, 1) == static_cast<int>(gridDim.x) - 1) {
      *done = 0;
      __threadfence_system();
      *reinterpret_cast<volatile unsigned*>(ready) = seq;
    }
  };
  if (id >= 2 * T) {
    __shared__ long long s_c[256];
    const int i = id - 2 * T;
    long long c = 0;
    for (int64_t k = tid; k < nblk; k += 256) c += cnt[i * nblk + k];
    s_c[tid] = c;
    __syncthreads();
    for (int o = 128; o > 0; o >>= 1) {
      if (tid < o) s_c[tid] += s_c[tid + o];
      __syncthreads();
    }
    if (tid == 0) out->count[i] = s_c[0];
    publish();
    return;
  }
  const int w = id / T, i = id % T;
  const double* src = part + (w * kMaxProbes + i) * nblk;
  if (SMEM) {
    extern __shared__ double s_tree[];
    const double v = tree_sum_smem(src, nblk, s_tree, tid, 256);
    if (tid == 0) (w == 0 ? out->err_sum : out->est_sum)[i] = v;
    publish();
    return;
  }
  double* bufs[2] = {scratch + static_cast<int64_t>(id) * 2 * nblk,
                     scratch + static_cast<int64_t>(id) * 2 * nblk + nblk};
  int cur_buf = 0;
  int64_t cur = nblk;
  while (cur > 1) {
    const int64_t half = cur / 2;
    double* dst = bufs[cur_buf];
    for (int64_t k = tid; k < half; k += 256) dst[k] = P_ADD(src[2 * k], src[2 * k + 1]);
    if ((cur & 1) && tid == 0) dst[half] = src[cur - 1];
    __syncthreads();
    src = dst;
    cur_buf ^= 1;
    cur = half + (cur & 1);
  }
  if (tid == 0) (w == 0 ? out->err_sum : out->est_sum)[i] = nblk ? src[0] : 0.0;
  publish();
}

// Exclusive block scan of one int64 per thread (NT = 1024 threads): warp
// shuffles, the 32 warp totals scanned by warp 0 -- two barriers instead of
// the 20 of a shared-memory Hillis-Steele scan.  `s` >= 33 entries; returns
// the thread's exclusive prefix, *total the block's sum.
__device__ __forceinline__ int64_t block_excl_scan_1024(int64_t local, int64_t* s,
                                                        int64_t* total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int64_t incl = local;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int64_t v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  if (lane == 31) s[w] = incl;
  __syncthreads();
  if (w == 0) {
    const int64_t x = s[lane];
    int64_t y = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t v = __shfl_up_sync(0xffffffffu, y, o);
      if (lane >= o) y += v;
    }
    s[lane] = y - x;
    if (lane == 31) s[32] = y;
  }
  __syncthreads();
  *total = s[32];
  return s[w] + incl - local;
}

// Exclusive scan of one count row (offsets of the accepted probe).
__global__ void __launch_bounds__(1024) k_scan_counts(int64_t nblk, const int64_t* cnt,
                                                      int64_t* offsets) {
  __shared__ int64_t s_sum[1024];
  const int tid = threadIdx.x;
  const int64_t chunk = (nblk + 1023) / 1024;
  const int64_t lo = tid * chunk, hi = lo + chunk < nblk ? lo + chunk : nblk;
  int64_t local = 0;
  for (int64_t i = lo; i < hi; ++i) local += cnt[i];
  int64_t total;
  int64_t run = block_excl_scan_1024(local, s_sum, &total);
  for (int64_t i = lo; i < hi; ++i) {
    offsets[i] = run;
    run += cnt[i];
  }
}

__global__ void k_candidates(int64_t m, double t, const uint8_t* flag, const double* err,
                             uint8_t* out) {
  const int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j < m) out[j] = (flag[j] && !(err[j] < t)) ? 1 : 0;
}

__global__ void k_fold_one(int64_t m, int64_t nblk, const double* __restrict__ x,
                           const uint8_t* __restrict__ flag, int which, double* part,
                           int64_t* cnt) {
  const int64_t b = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (b >= nblk) return;
  const int64_t lo = b * kBlock, hi = lo + kBlock < m ? lo + kBlock : m;
  int64_t other = 0;
  const double s = flag ? serial_fold<true>(x, flag, static_cast<uint8_t>(which), lo, hi, &other)
                        : serial_fold<false>(x, nullptr, 0, lo, hi, nullptr);
  part[b] = s;
  if (cnt) cnt[b] = (hi - lo) - other;  // entries equal to `which`
}

// ---- pairwise tree + offsets (single CTA) -----------------------------------
constexpr int kFinThreads = 1024;


// Zero-copy hand-off of the per-iteration scalars: `out` lives in mapped
// pinned host memory; the threads that wrote a field of it (tid 0: min/max,
// tid % 256 == 0: the tree sums, the last thread: the count) fence their
// writes at system scope, then one thread publishes the sequence number the
// host is spinning on.
// seq == 0: fence only (a later kernel publishes).
__device__ __forceinline__ void signal_host(unsigned* ready, unsigned seq) {
  if (!ready) return;
  if ((threadIdx.x & 255) == 0 || threadIdx.x == blockDim.x - 1) __threadfence_system();
  if (seq == 0) return;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    *reinterpret_cast<volatile unsigned*>(ready) = seq;
  }
}

// prepare_probes on the device: the same sorted thresholds / positions
// (insertion sort; the order among equal thresholds differs from std::sort's
// but equal thresholds have the same candidates, so every code test agrees).
__device__ void prepare_probes_dev(ProbeSet& ps) {
  int idx[kMaxProbes];
  int nn = 0, nf = 0;
  for (int j = 0; j < ps.T; ++j)
    if (ps.t[j] != ps.t[j]) ps.pos[j] = nn++;
  for (int j = 0; j < ps.T; ++j)
    if (ps.t[j] == ps.t[j]) {
      int k = nf++;
      while (k > 0 && ps.t[j] < ps.t[idx[k - 1]]) {
        idx[k] = idx[k - 1];
        --k;
      }
      idx[k] = j;
    }
  const double qnan = __longlong_as_double(0x7ff8000000000000LL);
  for (int k = 0; k < 16; ++k) ps.s[k] = k < nf ? ps.t[idx[k]] : qnan;
  for (int k = 0; k < nf; ++k) ps.pos[idx[k]] = nn + k;
  ps.nan_cnt = nn;
}

template <bool SMEM>
__global__ void __launch_bounds__(kFinThreads)
    k_finalize(int64_t nblk, int nq, const double* part, const int64_t* cnt, int64_t* offsets,
               double* scratch, FoldScalars* out, const unsigned long long* mm,
               const double* err0, unsigned* ready, unsigned seq, SpecProbe spec) {
  __shared__ double s_res[3];  // sum err, min, max (for the speculative first pass)
  extern __shared__ double s_tree[];
  __shared__ int64_t s_sum[kFinThreads];
  __shared__ unsigned long long s_k[2][kFinThreads / 32];
  const int tid = threadIdx.x;
  pdl_wait();  // the block records of the kernel before (launch_pdl)
  if (mm) {  // min_max of the errors from per-block keys (reduce.cpp:74-82; exact)
    unsigned long long a = ~0ULL, z = 0ULL;
    for (int64_t b0 = 0; b0 < nblk; b0 += 4 * kFinThreads) {  // 4 key pairs in flight
      ulonglong2 kk[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int64_t i = b0 + tid + static_cast<int64_t>(u) * kFinThreads;
        kk[u] = i < nblk ? reinterpret_cast<const ulonglong2*>(mm)[i] : make_ulonglong2(~0ULL, 0ULL);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        a = kk[u].x < a ? kk[u].x : a;
        z = kk[u].y > z ? kk[u].y : z;
      }
    }
    for (int o = 16; o > 0; o >>= 1) {
      const unsigned long long a2 = __shfl_xor_sync(0xffffffffu, a, o);
      const unsigned long long z2 = __shfl_xor_sync(0xffffffffu, z, o);
      a = a2 < a ? a2 : a;
      z = z2 > z ? z2 : z;
    }
    if ((tid & 31) == 0) {
      s_k[0][tid >> 5] = a;
      s_k[1][tid >> 5] = z;
    }
    __syncthreads();
    if (tid == 0) {
      for (int q = 1; q < kFinThreads / 32; ++q) {
        a = s_k[0][q] < a ? s_k[0][q] : a;
        z = s_k[1][q] > z ? s_k[1][q] : z;
      }
      const double x0 = err0[0];
      if (x0 != x0) {  // both start at x[0]; a NaN there sticks
        out->mn = x0;
        out->mx = x0;
      } else {
        out->mn = key_val(a);
        out->mx = key_val(z);
      }
      s_res[1] = out->mn;
      s_res[2] = out->mx;
    }
  }
  // reduce.cpp:13-27: p[i] = p[2i] + p[2i+1] level by level, odd tail carried.
  if constexpr (SMEM) {  // the nq <= 4 trees side by side, one 256-thread group each
    constexpr int G = kFinThreads / 4;
    const int q = tid / G;
    const double v = tree_sum_smem(part + (q < nq ? q : 0) * nblk, nblk,
                                   s_tree + q * (nblk + 64), tid % G, G);
    if (q < nq && tid % G == 0) out->sum[q] = v;
    if (q == 1 && tid % G == 0) s_res[0] = v;
    __syncthreads();
  } else
  for (int q = 0; q < nq; ++q) {
    const double* src = part + q * nblk;
    double* bufs[2] = {scratch, scratch + nblk};
    int cur_buf = 0;
    int64_t cur = nblk;
    while (cur > 1) {
      const int64_t half = cur / 2;
      double* dst = bufs[cur_buf];
      for (int64_t i = tid; i < half; i += kFinThreads) dst[i] = P_ADD(src[2 * i], src[2 * i + 1]);
      if ((cur & 1) && tid == 0) dst[half] = src[cur - 1];
      __syncthreads();
      src = dst;
      cur_buf ^= 1;
      cur = half + (cur & 1);
    }
    if (tid == 0) out->sum[q] = nblk ? src[0] : 0.0;
    if (tid == 0 && q == 1) s_res[0] = nblk ? src[0] : 0.0;
    __syncthreads();
  }
  if (!cnt) {
    if (tid == 0) out->count = 0;
    signal_host(ready, seq);
    return;
  }
  // exclusive scan of per-block counts (exact integers)
  const int64_t chunk = (nblk + kFinThreads - 1) / kFinThreads;
  const int64_t lo = tid * chunk, hi = lo + chunk < nblk ? lo + chunk : nblk;
  int64_t local = 0;
#pragma unroll 4
  for (int64_t i = lo; i < hi; ++i) local += cnt[i];
  static_assert(kFinThreads == 1024, "block_excl_scan_1024");
  int64_t total;
  int64_t run = block_excl_scan_1024(local, s_sum, &total);
  if (offsets)
    for (int64_t i = lo; i < hi; ++i) {
      offsets[i] = run;
      run += cnt[i];
    }
  if (tid == kFinThreads - 1) out->count = total;
  signal_host(ready, seq);
  if (spec.dev && mm && tid == 0) {
    // after the host has its scalars: the next search's first pass, built
    // from this iteration's e (the block-tree sum of the errors), batch size
    // and error min / max exactly as device_threshold builds it on the host
    ProbeSet ps{};
    build_probe_tree(ps, P_DIV(s_res[0], static_cast<double>(spec.s_it)), s_res[1], s_res[2]);
    prepare_probes_dev(ps);
    *spec.dev = ps;
  }
}

// ---- min / max ---------------------------------------------------------------
__global__ void k_minmax_init(unsigned long long* keys) {
  keys[0] = ~0ULL;
  keys[1] = 0ULL;
}

__global__ void k_minmax(int64_t m, const double* __restrict__ x, unsigned long long* keys) {
  unsigned long long lo = ~0ULL, hi = 0ULL;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < m;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const double v = __ldg(x + i);
    if (v != v) continue;  // NaN never wins a comparison (reduce.cpp:77-78)
    const unsigned long long k = ord_key(v);
    lo = k < lo ? k : lo;
    hi = k > hi ? k : hi;
  }
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long l2 = __shfl_xor_sync(0xffffffffu, lo, o);
    const unsigned long long h2 = __shfl_xor_sync(0xffffffffu, hi, o);
    lo = l2 < lo ? l2 : lo;
    hi = h2 > hi ? h2 : hi;
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMin(keys, lo);
    atomicMax(keys + 1, hi);
  }
}

__global__ void k_minmax_done(int64_t m, const double* x, const unsigned long long* keys,
                              double* out) {
  // reduce.cpp:75-76: both start at x[0]; a NaN there sticks.
  const double x0 = m ? x[0] : 0.0;
  if (m == 0 || x0 != x0) {
    out[0] = x0;
    out[1] = x0;
    return;
  }
  out[0] = key_val(keys[0]);
  out[1] = key_val(keys[1]);
}

// ---- fused filter + bisect ---------------------------------------------------
#ifndef PGN_SPLIT_THREADS
#define PGN_SPLIT_THREADS 512  // 4 rounds per 2048-block; 256 left a 2.35-wave tail (-10% at 512)
#endif
constexpr int kSplitThreads = PGN_SPLIT_THREADS;
constexpr int kSplitPer = static_cast<int>(kBlock) / kSplitThreads;  // 8

// Rank of each kept region inside its 2048-block: warp ballots + CTA scan.
__device__ __forceinline__ int64_t cta_rank(bool keep, int r, int64_t& carry, int* s_warp) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const unsigned bal = __ballot_sync(0xffffffffu, keep);
  const int before = __popc(bal & ((1u << lane) - 1u));
  if (lane == 0) s_warp[wid] = __popc(bal);
  __syncthreads();
  int wbase = 0, total = 0;
#pragma unroll
  for (int w = 0; w < kSplitThreads / 32; ++w) {
    const int c = s_warp[w];
    wbase += w < wid ? c : 0;
    total += c;
  }
  __syncthreads();
  const int64_t rank = carry + wbase + before;
  carry += total;
  (void)r;
  return rank;
}

__global__ void __launch_bounds__(kSplitThreads)
    k_split(int n, int64_t m, int64_t cap_src, int64_t cap_stage, const uint8_t* __restrict__ flag,
            int use_t, double t, const int64_t* __restrict__ offsets, const double* __restrict__ est,
            const double* __restrict__ err, const uint8_t* __restrict__ axis,
            const double* __restrict__ low, const double* __restrict__ len, double* dlow0,
            double* dlen0, double* dpest0, double* dperr, int64_t kbase, SplitWindow win) {
  __shared__ int s_warp[kSplitThreads / 32];
  const int64_t b = blockIdx.x;
  const int64_t base = b * kBlock;
  int64_t carry = offsets ? offsets[b] : base;
  for (int r = 0; r < kSplitPer; ++r) {
    const int64_t j = base + r * kSplitThreads + threadIdx.x;
    bool keep = j < m && (flag ? __ldg(flag + j) != 0 : true);
    if (use_t && keep) keep = !(__ldg(err + j) < t);  // accepted threshold (classify.cpp:63-66)
    const int64_t k = cta_rank(keep, r, carry, s_warp);
    if (!keep) continue;
    const int ax = __ldg(axis + j);
    int64_t c0 = 2 * (k - kbase);
    double *dlow = dlow0, *dlen = dlen0, *dpest = dpest0;
    int64_t cap_dst = cap_stage;
    if (win.low && c0 >= win.lo && c0 < win.hi) {  // stays on this rank: straight to the batch
      dlow = win.low, dlen = win.len, dpest = win.pest, cap_dst = win.cap;
      c0 += win.dst - win.lo;
    }
    for (int a = 0; a < n; ++a) {  // geometry.cpp:122-141
      const double lo = __ldg(low + a * cap_src + j);
      const double ln = __ldg(len + a * cap_src + j);
      double2 cl, cn;
      if (a == ax) {
        const double half = P_MUL(ln, 0.5);
        cl = make_double2(lo, P_ADD(lo, half));
        cn = make_double2(half, half);
      } else {
        cl = make_double2(lo, lo);
        cn = make_double2(ln, ln);
      }
      *reinterpret_cast<double2*>(dlow + a * cap_dst + c0) = cl;
      *reinterpret_cast<double2*>(dlen + a * cap_dst + c0) = cn;
    }
    const double e = __ldg(est + j);
    *reinterpret_cast<double2*>(dpest + c0) = make_double2(e, e);
    if (dperr) {
      const double r2 = __ldg(err + j);
      *reinterpret_cast<double2*>(dperr + c0) = make_double2(r2, r2);
    }
  }
}

__global__ void __launch_bounds__(kSplitThreads)
    k_compact(int n, int64_t m, int64_t cap, const uint8_t* __restrict__ flag,
              const int64_t* __restrict__ offsets, const double* low, const double* len,
              const double* est, const double* err, const int32_t* axis, const double* pest,
              const double* perr, double* klow, double* klen, double* kest, double* kerr,
              int32_t* kaxis, double* kpest, double* kperr) {
  __shared__ int s_warp[kSplitThreads / 32];
  const int64_t b = blockIdx.x;
  const int64_t base = b * kBlock;
  int64_t carry = offsets[b];
  for (int r = 0; r < kSplitPer; ++r) {
    const int64_t j = base + r * kSplitThreads + threadIdx.x;
    const bool keep = j < m && flag[j] != 0;
    const int64_t k = cta_rank(keep, r, carry, s_warp);
    if (!keep) continue;
    for (int a = 0; a < n; ++a) {
      klow[a * cap + k] = low[a * cap + j];
      klen[a * cap + k] = len[a * cap + j];
    }
    kest[k] = est[j];
    kerr[k] = err[j];
    kaxis[k] = axis[j];
    kpest[k] = pest[j];
    kperr[k] = perr[j];
  }
}

// ---- batch-API elementwise kernels -------------------------------------------
__global__ void k_refine(int64_t m, const double* est, const double* raw, const double* pest,
                         double* out) {
  const int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= m) return;
  const int64_t s = j ^ 1;  // errorest.cpp:24-36
  const double pair = P_ADD(raw[j], raw[s]);
  if (pair == 0.0 || !pgn_isfinite(pair)) {
    out[j] = raw[j];
    return;
  }
  const double delta = pgn_fabs(P_SUB(pest[j], P_ADD(est[j], est[s])));
  const double r = P_DIV(delta, pair);
  const double scale = r < 0.125 ? 0.125 : (1.0 < r ? 1.0 : r);
  out[j] = P_MUL(raw[j], scale);
}

__global__ void k_classify(int64_t m, const double* est, const double* err, double tau,
                           int enabled, uint8_t* flags) {
  const int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= m) return;
  if (!enabled) {
    flags[j] = 1;
    return;
  }
  const bool fin = est[j] == 0.0 ? err[j] == 0.0 : err[j] <= P_MUL(pgn_fabs(est[j]), tau);
  flags[j] = fin ? 0 : 1;
}

__global__ void k_apply_threshold(int64_t m, const double* err, double t, uint8_t* flags) {
  const int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j < m) flags[j] = err[j] < t ? 0 : 1;  // classify.cpp:29-35
}

// Naive serial volume sum (geometry.cpp:48-52 / classify.cpp:128-131), for
// the validation-only quantities.  One thread: it must be serial to match.
__global__ void k_serial_volume(int n, int64_t m, int64_t cap, const double* len,
                                const uint8_t* flag, int which, double* out) {
  double s = 0.0;
  for (int64_t j = 0; j < m; ++j) {
    if (flag && flag[j] != which) continue;
    double v = 1.0;
    for (int a = 0; a < n; ++a) v = P_MUL(v, len[a * cap + j]);
    s = P_ADD(s, v);
  }
  *out = s;
}

// validate_invariants: the kept regions' estimates in compacted order, summed
// serially inside 2048-element blocks of that order (reduce.cpp:13-27's
// leaves; the tree runs in k_finalize).  Debug path: one thread.
__global__ void k_kept_partials(int64_t m, const uint8_t* flag, int use_t, double t,
                                const double* err, const double* est, double* part) {
  double s = 0.0;
  int64_t c = 0;
  for (int64_t j = 0; j < m; ++j) {
    if (!flag[j] || (use_t && err[j] < t)) continue;
    s = P_ADD(s, est[j]);
    if (++c % kBlock == 0) {
      part[c / kBlock - 1] = s;
      s = 0.0;
    }
  }
  if (c % kBlock) part[c / kBlock] = s;
}

__global__ void k_math(int which, int64_t m, const double* x, double* y) {
  __shared__ __align__(16) uint64_t s_exp[256];
  __shared__ __align__(16) double s_sc[440];
  load_tables(s_exp, s_sc, g_exp_tab, reinterpret_cast<const double*>(g_sincos_tab));
  const int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= m) return;
  // the evaluator's hot-path variants (tab_exp / tab_cos: shared-address
  // tables, sign-bit XORs) and the branch-free cos
  const MathTables T = make_tables(s_exp, s_sc);
  if (which >= 3) {  // the paired forms the evaluator uses: (x[2i], x[2i+1]) as one pair
    const int64_t j0 = j & ~int64_t{1}, j1 = (j | 1) < m ? (j | 1) : j0;
    double ya, yb;
    if (which == 3)
      tab_exp2(x[j0], x[j1], T, ya, yb);
    else
      tab_cos2(x[j0], x[j1], T, ya, yb);
    y[j] = (j & 1) ? yb : ya;
    return;
  }
  y[j] = which == 0 ? tab_exp(x[j], T) : (which == 1 ? tab_cos(x[j], T) : gm_cos_bf(x[j], s_sc));
}

template <class F>
__global__ void k_call(int n, int64_t m, const double* x, IntegrandParams ip, double* y) {
  __shared__ __align__(16) uint64_t s_exp[256];
  __shared__ __align__(16) double s_sc[440];
  load_tables(s_exp, s_sc, g_exp_tab, reinterpret_cast<const double*>(g_sincos_tab));
  const int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= m) return;
  const MathTables T = make_tables(s_exp, s_sc);
  double xx[16];
  for (int a = 0; a < n; ++a) xx[a] = x[j * n + a];
  y[j] = eval_point<F>(xx, n, ip, T);
}

}  // namespace

namespace {

__global__ void k_pack_blocks(int64_t nblk_local, int64_t nblk_max, const double* part,
                              const int64_t* cnt, const unsigned long long* mm, const double* err,
                              BlockRec* recs) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i == 0) {
    BlockRec h{};
    h.part[0] = nblk_local > 0 ? err[0] : 0.0;
    h.cnt = nblk_local;
    recs[0] = h;
  }
  if (i >= nblk_max) return;
  BlockRec r{};
  if (i < nblk_local) {
    for (int q = 0; q < 4; ++q) r.part[q] = part[q * nblk_local + i];
    r.cnt = cnt[i];
    r.mn = mm[2 * i];
    r.mx = mm[2 * i + 1];
  }
  recs[1 + i] = r;
}

__global__ void k_unpack_blocks(RankBlocks rb, int64_t nblk_max, int64_t nblk_global,
                                const BlockRec* all, double* part, int64_t* cnt,
                                unsigned long long* mm, double* err0) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i == 0) {  // err[0] of the global batch: the first rank owning blocks
    for (int r = 0; r < rb.R; ++r)
      if (rb.nblk[r] > 0) {
        *err0 = all[r * (nblk_max + 1)].part[0];
        break;
      }
  }
  for (int r = 0; r < rb.R; ++r) {
    if (i >= rb.nblk[r]) continue;
    const BlockRec& x = all[r * (nblk_max + 1) + 1 + i];
    const int64_t g = rb.first[r] + i;
    for (int q = 0; q < 4; ++q) part[q * nblk_global + g] = x.part[q];
    cnt[g] = x.cnt;
    mm[2 * g] = x.mn;
    mm[2 * g + 1] = x.mx;
  }
}

__global__ void k_pack_probe(int64_t nblk_local, int64_t nblk_max, int T, const double* part,
                             const int64_t* cnt, ProbeRec* recs) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= nblk_max) return;
  ProbeRec r{};
  if (i < nblk_local)
    for (int k = 0; k < T; ++k) {
      r.err_sum[k] = part[(0 * kMaxProbes + k) * nblk_local + i];
      r.est_sum[k] = part[(1 * kMaxProbes + k) * nblk_local + i];
      r.cnt[k] = cnt[k * nblk_local + i];
    }
  recs[i] = r;
}

__global__ void k_unpack_probe(RankBlocks rb, int64_t nblk_max, int64_t nblk_global, int T,
                               const ProbeRec* all, double* part, int64_t* cnt) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  for (int r = 0; r < rb.R; ++r) {
    if (i >= rb.nblk[r]) continue;
    const ProbeRec& x = all[r * nblk_max + i];
    const int64_t g = rb.first[r] + i;
    for (int k = 0; k < T; ++k) {
      part[(0 * kMaxProbes + k) * nblk_global + g] = x.err_sum[k];
      part[(1 * kMaxProbes + k) * nblk_global + g] = x.est_sum[k];
      cnt[k * nblk_global + g] = x.cnt[k];
    }
  }
}

__global__ void k_gather_bounds(RankBlocks rb, const int64_t* offsets, const int64_t* cnt,
                                int64_t nblk_global, int64_t* out, unsigned* ready,
                                unsigned seq) {
  const int r = threadIdx.x;
  if (r < rb.R) out[r] = rb.first[r] < nblk_global ? offsets[rb.first[r]]
                                                    : (nblk_global ? offsets[nblk_global - 1] +
                                                                         cnt[nblk_global - 1]
                                                                   : 0);
  if (r == rb.R) out[r] = nblk_global ? offsets[nblk_global - 1] + cnt[nblk_global - 1] : 0;
  if (ready) {  // `out` is mapped host memory: fence every write, then publish
    if (r <= rb.R) __threadfence_system();
    __syncthreads();
    if (r == 0) {
      __threadfence_system();
      *reinterpret_cast<volatile unsigned*>(ready) = seq;
    }
  }
}

}  // namespace

void launch_pack_blocks(cudaStream_t st, int64_t nblk_local, int64_t nblk_max, const double* part,
                        const int64_t* cnt, const unsigned long long* mm, const double* err,
                        BlockRec* recs) {
  const int64_t w = nblk_max > 0 ? nblk_max : 1;
  k_pack_blocks<<<grid_for(w, 256), 256, 0, st>>>(nblk_local, nblk_max, part, cnt, mm, err, recs);
}
void launch_unpack_blocks(cudaStream_t st, const RankBlocks& rb, int64_t nblk_max,
                          int64_t nblk_global, const BlockRec* all, double* part, int64_t* cnt,
                          unsigned long long* mm, double* err0) {
  const int64_t w = nblk_max > 0 ? nblk_max : 1;
  k_unpack_blocks<<<grid_for(w, 256), 256, 0, st>>>(rb, nblk_max, nblk_global, all, part, cnt, mm,
                                                    err0);
}
void launch_pack_probe(cudaStream_t st, int64_t nblk_local, int64_t nblk_max, int T,
                       const double* part, const int64_t* cnt, ProbeRec* recs) {
  if (nblk_max > 0)
    k_pack_probe<<<grid_for(nblk_max, 128), 128, 0, st>>>(nblk_local, nblk_max, T, part, cnt, recs);
}
void launch_unpack_probe(cudaStream_t st, const RankBlocks& rb, int64_t nblk_max,
                         int64_t nblk_global, int T, const ProbeRec* all, double* part,
                         int64_t* cnt) {
  if (nblk_max > 0)
    k_unpack_probe<<<grid_for(nblk_max, 128), 128, 0, st>>>(rb, nblk_max, nblk_global, T, all,
                                                            part, cnt);
}
void launch_gather_bounds(cudaStream_t st, const RankBlocks& rb, const int64_t* offsets,
                          const int64_t* cnt, int64_t nblk_global, int64_t* out, unsigned* ready,
                          unsigned seq) {
  k_gather_bounds<<<1, kMaxRanks + 1, 0, st>>>(rb, offsets, cnt, nblk_global, out, ready, seq);
}

const uint64_t* device_exp_table() {
  void* p = nullptr;
  cudaGetSymbolAddress(&p, g_exp_tab);
  return static_cast<const uint64_t*>(p);
}
const double* device_sincos_table() {
  void* p = nullptr;
  cudaGetSymbolAddress(&p, g_sincos_tab);
  return static_cast<const double*>(p);
}

void launch_uniform_split(cudaStream_t st, int n, int d, int64_t m, int64_t cap, double* low,
                          double* len, const double* lower, const double* step, int64_t first) {
  if (m <= 0) return;
  k_uniform_split<<<grid_for(m, 256), 256, 0, st>>>(n, d, m, cap, low, len, lower, step, first);
}

void launch_fold_eval(cudaStream_t st, int64_t m, const double* est, const double* err,
                      const uint8_t* flag, double* part, int64_t* cnt, int use_t, double t) {
  const int64_t nblk = nblocks_of(m);
  if (nblk == 0) return;
  k_fold_eval<<<static_cast<unsigned>(nblk), kFoldThreads, 0, st>>>(m, nblk, est, err, flag,
                                                                     part, cnt, use_t, t);
}


bool pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("PAGANI_PDL");
    return !e || std::atoi(e) != 0;
  }();
  return on;
}

// Opt a kernel in to > 48 KB of dynamic shared memory, once per (device, kernel).
void opt_in_smem(const void* fn) {
  static std::mutex mu;
  static std::set<std::pair<int, const void*>> done;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> g(mu);
  if (done.insert({dev, fn}).second)
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(kTreeSmemMaxBytes));
}

void finalize_multi(cudaStream_t st, int64_t nblk, int T, const double* part,
                    const int64_t* cnt, double* scratch, ProbeScalars* out, unsigned* ready,
                    unsigned seq, int* done) {
  const size_t sm = tree_smem_bytes(nblk, 1);
  if (sm <= static_cast<size_t>(kTreeSmemMaxBytes)) {
    opt_in_smem(reinterpret_cast<const void*>(&k_finalize_multi<true>));
    (void)(launch_pdl(&k_finalize_multi<true>, dim3(3 * T), dim3(256), sm, st, nblk, T, part, cnt,
                      scratch, out, ready, seq, done));
  } else {
    (void)(launch_pdl(&k_finalize_multi<false>, dim3(3 * T), dim3(256), 0, st, nblk, T, part, cnt,
                      scratch, out, ready, seq, done));
  }
}

void prepare_probes(ProbeSet& ps) {
  int idx[kMaxProbes];
  int nn = 0, nf = 0;
  for (int j = 0; j < ps.T; ++j)
    if (ps.t[j] != ps.t[j]) ps.pos[j] = nn++;
  for (int j = 0; j < ps.T; ++j)
    if (ps.t[j] == ps.t[j]) idx[nf++] = j;
  std::sort(idx, idx + nf, [&](int a, int b) { return ps.t[a] < ps.t[b]; });
  const double qnan = std::numeric_limits<double>::quiet_NaN();
  for (int k = 0; k < 16; ++k) ps.s[k] = k < nf ? ps.t[idx[k]] : qnan;
  for (int k = 0; k < nf; ++k) ps.pos[idx[k]] = nn + k;
  ps.nan_cnt = nn;
}

void launch_probe_only(cudaStream_t st, int64_t m, const ProbeSet& ts, const double* est,
                       const double* err, const uint8_t* flag, double* part, int64_t* cnt) {
  const int64_t nblk = nblocks_of(m);
  if (nblk == 0) return;
  k_probe_multi<<<static_cast<unsigned>(nblk), kProbeThreads, 0, st>>>(m, nblk, ts, est, err,
                                                                        flag, part, cnt, nullptr);
}

void launch_finalize_multi(cudaStream_t st, int64_t nblk, int T, const double* part,
                           const int64_t* cnt, double* scratch, ProbeScalars* out,
                           unsigned* ready, unsigned seq, int* done) {
  finalize_multi(st, nblk, T, part, cnt, scratch, out, ready, seq, done);
}

void launch_probe_multi(cudaStream_t st, int64_t m, const ProbeSet& ts, const double* est,
                        const double* err, const uint8_t* flag, double* part, int64_t* cnt,
                        double* scratch, ProbeScalars* out, unsigned* ready, unsigned seq,
                        int* done) {
  const int64_t nblk = nblocks_of(m);
  if (nblk == 0) return;
  k_probe_multi<<<static_cast<unsigned>(nblk), kProbeThreads, 0, st>>>(m, nblk, ts, est, err,
                                                                        flag, part, cnt, nullptr);
  finalize_multi(st, nblk, ts.T, part, cnt, scratch, out, ready, seq, done);
}

void launch_probe_multi_dev(cudaStream_t st, int64_t m, const ProbeSet* dts, const double* est,
                            const double* err, const uint8_t* flag, double* part, int64_t* cnt,
                            double* scratch, ProbeScalars* out, unsigned* ready, unsigned seq,
                            int* done) {
  const int64_t nblk = nblocks_of(m);
  if (nblk == 0) return;
  (void)(launch_pdl(&k_probe_multi, dim3(static_cast<unsigned>(nblk)), dim3(kProbeThreads), 0, st,
                    m, nblk, ProbeSet{}, est, err, flag, part, cnt, dts));
  finalize_multi(st, nblk, kMaxProbes, part, cnt, scratch, out, ready, seq, done);
}

int probe_fast_grid(int64_t m) {
  const int64_t want = (m + 8 * kPfThreads - 1) / (8 * kPfThreads);  // >= 8 regions per thread
  const int64_t cap = 148 * 8;
  return static_cast<int>(want < 1 ? 1 : (want > cap ? cap : want));
}

void launch_probe_fast(cudaStream_t st, int64_t m, const ProbeSet& ts, const double* err,
                       const uint8_t* flag, double* part, int64_t* cnt, ProbeScalars* out,
                       unsigned* ready, unsigned seq) {
  const int G = probe_fast_grid(m);
  if (m > 0) k_probe_fast<<<G, kPfThreads, 0, st>>>(m, ts, err, flag, part, cnt);
  k_probe_fast_total<<<1, 512, 0, st>>>(m > 0 ? G : 0, part, cnt, out, ready, seq);
}

void launch_fold_threshold(cudaStream_t st, int64_t m, const double* est, const double* err,
                           const uint8_t* flag, double t, double* part, int64_t* cnt) {
  const int64_t nblk = nblocks_of(m);
  if (nblk > 0)
    k_fold_threshold<<<static_cast<unsigned>(nblk), kFtThreads, 0, st>>>(m, nblk, est, err, flag,
                                                                         t, part, cnt);
}

void launch_scan_counts(cudaStream_t st, int64_t nblk, const int64_t* cnt, int64_t* offsets) {
  if (nblk > 0) k_scan_counts<<<1, 1024, 0, st>>>(nblk, cnt, offsets);
}

void launch_candidates(cudaStream_t st, int64_t m, double t, const uint8_t* flag,
                       const double* err, uint8_t* out) {
  if (m > 0) k_candidates<<<grid_for(m, 256), 256, 0, st>>>(m, t, flag, err, out);
}

void launch_fold_one(cudaStream_t st, int64_t m, const double* x, const uint8_t* flag,
                     int which, double* part, int64_t* cnt) {
  const int64_t nblk = nblocks_of(m);
  if (nblk == 0) return;
  k_fold_one<<<grid_for(nblk, 128), 128, 0, st>>>(m, nblk, x, flag, which, part, cnt);
}

void launch_finalize(cudaStream_t st, int64_t nblk, int nq, const double* part,
                     const int64_t* cnt, int64_t* offsets, double* scratch, FoldScalars* out,
                     const unsigned long long* mm, const double* err0, unsigned* ready,
                     unsigned seq, const SpecProbe& spec) {
  const size_t sm = tree_smem_bytes(nblk, 4);
  if (sm <= static_cast<size_t>(kTreeSmemMaxBytes)) {
    opt_in_smem(reinterpret_cast<const void*>(&k_finalize<true>));
    (void)(launch_pdl(&k_finalize<true>, dim3(1), dim3(kFinThreads), sm, st, nblk, nq, part, cnt,
                      offsets, scratch, out, mm, err0, ready, seq, spec));
  } else {
    (void)(launch_pdl(&k_finalize<false>, dim3(1), dim3(kFinThreads), 0, st, nblk, nq, part, cnt,
                      offsets, scratch, out, mm, err0, ready, seq, spec));
  }
}

void launch_minmax(cudaStream_t st, int64_t m, const double* x, unsigned long long* keys,
                   double* out) {
  k_minmax_init<<<1, 1, 0, st>>>(keys);
  if (m > 0) {
    int blocks = static_cast<int>(grid_for(m, 256));
    if (blocks > 148 * 8) blocks = 148 * 8;
    k_minmax<<<blocks, 256, 0, st>>>(m, x, keys);
  }
  k_minmax_done<<<1, 1, 0, st>>>(m, x, keys, out);
}

// k_split_n<N>: the same fused filter + bisect as k_split with the dimension
// known at compile time, restructured for memory-level parallelism: every
// flag (and err) of the CTA's 8 rounds is loaded up front, the 8 rounds' ranks
// come from one shared-memory scan (one barrier instead of 16), and each kept
// region issues all 2N + 2 of its loads before any store.
template <int N>
__global__ void __launch_bounds__(kSplitThreads)
    k_split_n(int64_t m, int64_t cap_src, int64_t cap_stage, const uint8_t* __restrict__ flag,
              int use_t, double t, const int64_t* __restrict__ offsets,
              const double* __restrict__ est, const double* __restrict__ err,
              const uint8_t* __restrict__ axis, const double* __restrict__ low,
              const double* __restrict__ len, double* __restrict__ dlow0,
              double* __restrict__ dlen0, double* __restrict__ dpest0, double* __restrict__ dperr,
              int64_t kbase, SplitWindow win) {
  constexpr int W = kSplitThreads / 32;
  __shared__ int s_cnt[kSplitPer][W];
  const int64_t b = blockIdx.x;
  const int64_t base = b * kBlock;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  bool keep[kSplitPer];
  uint8_t fl[kSplitPer];
  double ev[kSplitPer];
#pragma unroll
  for (int r = 0; r < kSplitPer; ++r) {
    const int64_t j = base + r * kSplitThreads + threadIdx.x;
    fl[r] = j < m ? (flag ? __ldg(flag + j) : uint8_t{1}) : uint8_t{0};
    ev[r] = (use_t && j < m) ? __ldg(err + j) : 0.0;
  }
  unsigned before[kSplitPer];
#pragma unroll
  for (int r = 0; r < kSplitPer; ++r) {
    keep[r] = fl[r] != 0 && !(use_t && ev[r] < t);  // accepted threshold (classify.cpp:63-66)
    const unsigned bal = __ballot_sync(0xffffffffu, keep[r]);
    before[r] = __popc(bal & ((1u << lane) - 1u));
    if (lane == 0) s_cnt[r][wid] = __popc(bal);
  }
  __syncthreads();
  int64_t run = offsets ? offsets[b] : base;  // rank of the block's first kept region
#pragma unroll
  for (int r = 0; r < kSplitPer; ++r) {
    int wbase = 0, total = 0;
#pragma unroll
    for (int w = 0; w < W; ++w) {
      const int c = s_cnt[r][w];
      wbase += w < wid ? c : 0;
      total += c;
    }
    const int64_t k = run + wbase + before[r];
    run += total;
    if (!keep[r]) continue;
    const int64_t j = base + r * kSplitThreads + threadIdx.x;
    const int ax = __ldg(axis + j);
    const double e = __ldg(est + j);
    double lo[N], ln[N];
#pragma unroll
    for (int a = 0; a < N; ++a) {
      lo[a] = __ldg(low + a * cap_src + j);
      ln[a] = __ldg(len + a * cap_src + j);
    }
    int64_t c0 = 2 * (k - kbase);
    double *dlow = dlow0, *dlen = dlen0, *dpest = dpest0;
    int64_t cap_dst = cap_stage;
    if (win.low && c0 >= win.lo && c0 < win.hi) {  // stays on this rank: straight to the batch
      dlow = win.low, dlen = win.len, dpest = win.pest, cap_dst = win.cap;
      c0 += win.dst - win.lo;
    }
#pragma unroll
    for (int a = 0; a < N; ++a) {  // geometry.cpp:122-141
      double2 cl, cn;
      if (a == ax) {
        const double half = P_MUL(ln[a], 0.5);
        cl = make_double2(lo[a], P_ADD(lo[a], half));
        cn = make_double2(half, half);
      } else {
        cl = make_double2(lo[a], lo[a]);
        cn = make_double2(ln[a], ln[a]);
      }
      *reinterpret_cast<double2*>(dlow + a * cap_dst + c0) = cl;
      *reinterpret_cast<double2*>(dlen + a * cap_dst + c0) = cn;
    }
    *reinterpret_cast<double2*>(dpest + c0) = make_double2(e, e);
    if (dperr) {
      const double r2 = __ldg(err + j);
      *reinterpret_cast<double2*>(dperr + c0) = make_double2(r2, r2);
    }
  }
}

// ---- k_split_bulk<N>: the same fused filter + bisect, geometry staged by TMA --
// The kept regions' geometry is a sparse subset of the axis-major store, read
// at 32-byte sector granularity either way; this form reads each
// 2048-block's low/len rows densely with 1-D bulk copies (cp.async.bulk, 16 KB
// per row, completion on an mbarrier) into a 2-stage shared-memory ring -- one
// axis per stage, the next axis in flight while the current one is written --
// so the loads never occupy registers or warps.  Threads then build the child
// pairs of their kept regions from shared memory and store them coalesced.
// Blocks without a kept region issue no copies.  Used when most regions are
// kept (the host picks it by the kept fraction); k_split_n otherwise.
constexpr int kBulkThreads = 256;
constexpr int kBulkPer = static_cast<int>(kBlock) / kBulkThreads;  // 8 rounds
constexpr size_t kBulkSmem = 2 * 2 * kBlock * sizeof(double);     // 2 stages x {low, len}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  } while (!done);
}

template <int N>
__global__ void __launch_bounds__(kBulkThreads, 3)
    k_split_bulk(int64_t m, int64_t cap_src, int64_t cap_stage, const uint8_t* __restrict__ flag,
                 int use_t, double t, const int64_t* __restrict__ offsets, int64_t kept_end,
                 const double* __restrict__ est, const double* __restrict__ err,
                 const uint8_t* __restrict__ axis, const double* __restrict__ low,
                 const double* __restrict__ len, double* __restrict__ dlow0,
                 double* __restrict__ dlen0, double* __restrict__ dpest0, int64_t kbase,
                 SplitWindow win) {
  constexpr int W = kBulkThreads / 32;
  extern __shared__ __align__(128) double sbuf[];  // [stage][low | len][kBlock]
  __shared__ __align__(8) uint64_t bar[2];
  __shared__ int s_cnt[kBulkPer][W];
  const int64_t b = blockIdx.x;
  const int64_t base = b * kBlock;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int cnt = static_cast<int>(m - base < kBlock ? m - base : kBlock);
  // the block's kept count from the exclusive scan: blocks with none issue
  // no copies, the others start their first two rows before anything else
  const int64_t k_first = offsets[b];
  const int64_t k_next = b + 1 < static_cast<int64_t>(gridDim.x) ? offsets[b + 1] : kept_end;
  if (k_next == k_first) return;
  // rows are copied in 16-byte units; the store is allocated in 2048-blocks,
  // so rounding an odd count up stays inside it
  const uint32_t row_bytes = static_cast<uint32_t>(((cnt + 1) & ~1) * sizeof(double));
  auto issue = [&](int a, int st) {  // one thread: rows low[a], len[a] -> stage st
    mbar_expect_tx(&bar[st], 2 * row_bytes);
    bulk_g2s(sbuf + (2 * st) * kBlock, low + a * cap_src + base, row_bytes, &bar[st]);
    bulk_g2s(sbuf + (2 * st + 1) * kBlock, len + a * cap_src + base, row_bytes, &bar[st]);
  };
  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
#pragma unroll
    for (int st = 0; st < 2 && st < N; ++st) issue(st, st);
  }

  // ranks of the kept regions (as k_split_n)
  bool keep[kBulkPer];
  unsigned before[kBulkPer];
#pragma unroll
  for (int r = 0; r < kBulkPer; ++r) {
    const int i = r * kBulkThreads + tid;
    const int64_t j = base + i;
    const uint8_t fl = i < cnt ? (flag ? __ldg(flag + j) : uint8_t{1}) : uint8_t{0};
    const double ev = (use_t && i < cnt) ? __ldg(err + j) : 0.0;
    keep[r] = fl != 0 && !(use_t && ev < t);  // classify.cpp:63-66
    const unsigned bal = __ballot_sync(0xffffffffu, keep[r]);
    before[r] = __popc(bal & ((1u << lane) - 1u));
    if (lane == 0) s_cnt[r][wid] = __popc(bal);
  }
  __syncthreads();  // s_cnt and the barrier initialisation visible to all
  // child slots: c0 = 2 (k - kbase), routed to the next batch (window) or staging
  int64_t run = k_first;
  int64_t c0[kBulkPer];
  bool inwin[kBulkPer];
  uint32_t ax_pack[2] = {0u, 0u};
#pragma unroll
  for (int r = 0; r < kBulkPer; ++r) {
    int wbase = 0, tot = 0;
#pragma unroll
    for (int w = 0; w < W; ++w) {
      const int c = s_cnt[r][w];
      wbase += w < wid ? c : 0;
      tot += c;
    }
    const int64_t k = run + wbase + before[r];
    run += tot;
    int64_t c = 2 * (k - kbase);
    inwin[r] = win.low && c >= win.lo && c < win.hi;
    if (inwin[r]) c += win.dst - win.lo;
    c0[r] = c;
    if (keep[r]) {
      const int64_t j = base + r * kBulkThreads + tid;
      const double e = __ldg(est + j);
      double* dp = inwin[r] ? win.pest : dpest0;
      *reinterpret_cast<double2*>(dp + c) = make_double2(e, e);
      ax_pack[r >> 2] |= static_cast<uint32_t>(__ldg(axis + j)) << (8 * (r & 3));
    }
  }
#pragma unroll 1
  for (int a = 0; a < N; ++a) {
    const int st = a & 1;
    mbar_wait(&bar[st], static_cast<uint32_t>(a >> 1) & 1u);
    const double* sl = sbuf + (2 * st) * kBlock;
    const double* sn = sbuf + (2 * st + 1) * kBlock;
#pragma unroll
    for (int r = 0; r < kBulkPer; ++r) {
      if (!keep[r]) continue;
      const int i = r * kBulkThreads + tid;
      const double lo = sl[i], ln = sn[i];
      const int ax = static_cast<int>((ax_pack[r >> 2] >> (8 * (r & 3))) & 0xffu);
      double2 cl, cn;
      if (a == ax) {  // geometry.cpp:122-141
        const double half = P_MUL(ln, 0.5);
        cl = make_double2(lo, P_ADD(lo, half));
        cn = make_double2(half, half);
      } else {
        cl = make_double2(lo, lo);
        cn = make_double2(ln, ln);
      }
      double* dl = inwin[r] ? win.low : dlow0;
      double* dn = inwin[r] ? win.len : dlen0;
      const int64_t capd = inwin[r] ? win.cap : cap_stage;
      *reinterpret_cast<double2*>(dl + a * capd + c0[r]) = cl;
      *reinterpret_cast<double2*>(dn + a * capd + c0[r]) = cn;
    }
    if (a + 2 < N) {
      __syncthreads();  // every thread is done with stage st
      if (tid == 0) issue(a + 2, st);
    }
  }
}

// Persistent form of k_split_bulk (N >= 2): one CTA per resident slot, each
// walking the blocks b = blockIdx.x, + gridDim.x, ... that have kept
// regions.  The CTA's geometry rows form one stream g = 0, 1, 2, ... (row a
// of its i-th block is g = i N + a), staged through the same 2-slot ring
// (slot g & 1, mbarrier phase (g >> 1) & 1); a freed slot is refilled with row
// g + 2 -- for the last two rows of a block that is the next block's first
// two rows, so the next block's loads are in flight while this block is
// finished and the next block's flags are scanned, and there is no wave tail.
template <int N>
__global__ void __launch_bounds__(kBulkThreads, 3)
    k_split_bulk_p(int64_t m, int64_t nblk, int64_t cap_src, int64_t cap_stage,
                   const uint8_t* __restrict__ flag, int use_t, double t,
                   const int64_t* __restrict__ offsets, int64_t kept_end,
                   const double* __restrict__ est, const double* __restrict__ err,
                   const uint8_t* __restrict__ axis, const double* __restrict__ low,
                   const double* __restrict__ len, double* __restrict__ dlow0,
                   double* __restrict__ dlen0, double* __restrict__ dpest0, int64_t kbase,
                   SplitWindow win) {
  static_assert(N >= 2, "the persistent split streams two rows ahead within a block pair");
  constexpr int W = kBulkThreads / 32;
  extern __shared__ __align__(128) double sbuf[];  // [slot][low | len][kBlock]
  __shared__ __align__(8) uint64_t bar[2];
  __shared__ int s_cnt[kBulkPer][W];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  auto kfirst = [&](int64_t b) { return offsets[b]; };
  auto knext = [&](int64_t b) { return b + 1 < nblk ? offsets[b + 1] : kept_end; };
  auto next_block = [&](int64_t b) {  // the CTA's next block with kept regions
    while (b < nblk && knext(b) == kfirst(b)) b += gridDim.x;
    return b;
  };
  auto row_bytes = [&](int64_t b) {
    const int64_t c = m - b * kBlock < kBlock ? m - b * kBlock : kBlock;
    return static_cast<uint32_t>(((c + 1) & ~int64_t{1}) * sizeof(double));
  };
  auto issue = [&](int64_t b, int a, int slot) {  // one thread: rows low[a], len[a] of block b
    const uint32_t rb = row_bytes(b);
    mbar_expect_tx(&bar[slot], 2 * rb);
    bulk_g2s(sbuf + (2 * slot) * kBlock, low + a * cap_src + b * kBlock, rb, &bar[slot]);
    bulk_g2s(sbuf + (2 * slot + 1) * kBlock, len + a * cap_src + b * kBlock, rb, &bar[slot]);
  };
  int64_t b = next_block(blockIdx.x);
  if (b >= nblk) return;
  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    issue(b, 0, 0);
    issue(b, 1, 1);
  }
  uint32_t g = 0;  // global row counter of this CTA
  while (b < nblk) {
    const int64_t bn = next_block(b + gridDim.x);
    const int64_t base = b * kBlock;
    const int cnt = static_cast<int>(m - base < kBlock ? m - base : kBlock);
    bool keep[kBulkPer];
    unsigned before[kBulkPer];
#pragma unroll
    for (int r = 0; r < kBulkPer; ++r) {
      const int i = r * kBulkThreads + tid;
      const int64_t j = base + i;
      const uint8_t fl = i < cnt ? (flag ? __ldg(flag + j) : uint8_t{1}) : uint8_t{0};
      const double ev = (use_t && i < cnt) ? __ldg(err + j) : 0.0;
      keep[r] = fl != 0 && !(use_t && ev < t);  // classify.cpp:63-66
      const unsigned bal = __ballot_sync(0xffffffffu, keep[r]);
      before[r] = __popc(bal & ((1u << lane) - 1u));
      if (lane == 0) s_cnt[r][wid] = __popc(bal);
    }
    __syncthreads();
    int64_t run = kfirst(b);
    int64_t c0[kBulkPer];
    bool inwin[kBulkPer];
    uint32_t ax_pack[2] = {0u, 0u};
#pragma unroll
    for (int r = 0; r < kBulkPer; ++r) {
      int wbase = 0, tot = 0;
#pragma unroll
      for (int w = 0; w < W; ++w) {
        const int c = s_cnt[r][w];
        wbase += w < wid ? c : 0;
        tot += c;
      }
      const int64_t k = run + wbase + before[r];
      run += tot;
      int64_t c = 2 * (k - kbase);
      inwin[r] = win.low && c >= win.lo && c < win.hi;
      if (inwin[r]) c += win.dst - win.lo;
      c0[r] = c;
      if (keep[r]) {
        const int64_t j = base + r * kBulkThreads + tid;
        const double e = __ldg(est + j);
        double* dp = inwin[r] ? win.pest : dpest0;
        *reinterpret_cast<double2*>(dp + c) = make_double2(e, e);
        ax_pack[r >> 2] |= static_cast<uint32_t>(__ldg(axis + j)) << (8 * (r & 3));
      }
    }
#pragma unroll 1
    for (int a = 0; a < N; ++a, ++g) {
      const int slot = static_cast<int>(g & 1u);
      mbar_wait(&bar[slot], (g >> 1) & 1u);
      const double* sl = sbuf + (2 * slot) * kBlock;
      const double* sn = sbuf + (2 * slot + 1) * kBlock;
#pragma unroll
      for (int r = 0; r < kBulkPer; ++r) {
        if (!keep[r]) continue;
        const int i = r * kBulkThreads + tid;
        const double lo = sl[i], ln = sn[i];
        const int ax = static_cast<int>((ax_pack[r >> 2] >> (8 * (r & 3))) & 0xffu);
        double2 cl, cn;
        if (a == ax) {  // geometry.cpp:122-141
          const double half = P_MUL(ln, 0.5);
          cl = make_double2(lo, P_ADD(lo, half));
          cn = make_double2(half, half);
        } else {
          cl = make_double2(lo, lo);
          cn = make_double2(ln, ln);
        }
        double* dl = inwin[r] ? win.low : dlow0;
        double* dn = inwin[r] ? win.len : dlen0;
        const int64_t capd = inwin[r] ? win.cap : cap_stage;
        *reinterpret_cast<double2*>(dl + a * capd + c0[r]) = cl;
        *reinterpret_cast<double2*>(dn + a * capd + c0[r]) = cn;
      }
      __syncthreads();  // every thread is done with this slot (and with s_cnt)
      if (tid == 0) {   // refill it with the stream's row g + 2
        if (a + 2 < N)
          issue(b, a + 2, slot);
        else if (bn < nblk)
          issue(bn, a + 2 - N, slot);
      }
    }
    b = bn;
  }
}

// PAGANI_SPLIT_PERSISTENT=1 selects the persistent k_split_bulk_p (A/B:
// measured slower on B200 -- 112.4 vs 107.0 ms per bench step -- so the
// one-CTA-per-block form is the default).
static bool split_persistent() {
  static const bool on = [] {
    const char* e = std::getenv("PAGANI_SPLIT_PERSISTENT");
    return e && std::atoi(e) != 0;
  }();
  return on;
}

void launch_split(cudaStream_t st, int n, int64_t m, int64_t cap_src, int64_t cap_dst,
                  const uint8_t* flag, int use_t, double t, const int64_t* offsets,
                  const double* est,
                  const double* err, const uint8_t* axis, const double* low, const double* len,
                  double* dlow, double* dlen, double* dpest, double* dperr, int64_t kbase,
                  const SplitWindow& win, bool bulk, int64_t kept_end) {
  const int64_t nblk = nblocks_of(m);
  if (nblk == 0) return;
  const unsigned g = static_cast<unsigned>(nblk);
  if (bulk && offsets && kept_end >= 0 && !dperr && n >= 2 && n <= 16 && split_persistent()) {
    static int sms = [] {
      int d = 0, v = 148;
      cudaGetDevice(&d);
      cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, d);
      return v;
    }();
    const int64_t slots = static_cast<int64_t>(sms) * 3;
    const unsigned gp = static_cast<unsigned>(nblk < slots ? nblk : slots);
    switch (n) {
#define PGN_BULKP_CASE(NN)                                                                     \
  case NN:                                                                                     \
    opt_in_smem(reinterpret_cast<const void*>(&k_split_bulk_p<NN>));                          \
    k_split_bulk_p<NN><<<gp, kBulkThreads, kBulkSmem, st>>>(                                   \
        m, nblk, cap_src, cap_dst, flag, use_t, t, offsets, kept_end, est, err, axis, low, len, \
        dlow, dlen, dpest, kbase, win);                                                        \
    return;
      PGN_BULKP_CASE(2) PGN_BULKP_CASE(3) PGN_BULKP_CASE(4) PGN_BULKP_CASE(5)
      PGN_BULKP_CASE(6) PGN_BULKP_CASE(7) PGN_BULKP_CASE(8) PGN_BULKP_CASE(9) PGN_BULKP_CASE(10)
      PGN_BULKP_CASE(11) PGN_BULKP_CASE(12) PGN_BULKP_CASE(13) PGN_BULKP_CASE(14)
      PGN_BULKP_CASE(15) PGN_BULKP_CASE(16)
#undef PGN_BULKP_CASE
      default: break;
    }
  }
  if (bulk && offsets && kept_end >= 0 && !dperr && n >= 1 && n <= 16) {
    switch (n) {
#define PGN_BULK_CASE(NN)                                                                      \
  case NN: {                                                                                   \
    opt_in_smem(reinterpret_cast<const void*>(&k_split_bulk<NN>));                             \
    k_split_bulk<NN><<<g, kBulkThreads, kBulkSmem, st>>>(m, cap_src, cap_dst, flag, use_t, t,  \
                                                         offsets, kept_end, est, err, axis,    \
                                                         low, len, dlow, dlen, dpest, kbase,   \
                                                         win);                                 \
    return;                                                                                    \
  }
      PGN_BULK_CASE(1) PGN_BULK_CASE(2) PGN_BULK_CASE(3) PGN_BULK_CASE(4) PGN_BULK_CASE(5)
      PGN_BULK_CASE(6) PGN_BULK_CASE(7) PGN_BULK_CASE(8) PGN_BULK_CASE(9) PGN_BULK_CASE(10)
      PGN_BULK_CASE(11) PGN_BULK_CASE(12) PGN_BULK_CASE(13) PGN_BULK_CASE(14)
      PGN_BULK_CASE(15) PGN_BULK_CASE(16)
#undef PGN_BULK_CASE
      default: break;
    }
  }
  switch (n) {
#define PGN_SPLIT_CASE(NN)                                                                      \
  case NN:                                                                                      \
    k_split_n<NN><<<g, kSplitThreads, 0, st>>>(m, cap_src, cap_dst, flag, use_t, t, offsets, est, \
                                               err, axis, low, len, dlow, dlen, dpest, dperr,    \
                                               kbase, win);                                     \
    return;
    PGN_SPLIT_CASE(1) PGN_SPLIT_CASE(2) PGN_SPLIT_CASE(3) PGN_SPLIT_CASE(4) PGN_SPLIT_CASE(5)
    PGN_SPLIT_CASE(6) PGN_SPLIT_CASE(7) PGN_SPLIT_CASE(8) PGN_SPLIT_CASE(9) PGN_SPLIT_CASE(10)
    PGN_SPLIT_CASE(11) PGN_SPLIT_CASE(12) PGN_SPLIT_CASE(13) PGN_SPLIT_CASE(14)
    PGN_SPLIT_CASE(15) PGN_SPLIT_CASE(16)
#undef PGN_SPLIT_CASE
    default:
      k_split<<<g, kSplitThreads, 0, st>>>(n, m, cap_src, cap_dst, flag, use_t, t, offsets, est,
                                           err, axis, low, len, dlow, dlen, dpest, dperr, kbase,
                                           win);
  }
}

// ---- k_link: the filter half of k_split, bisection deferred into k_evaluate --
// Region j is kept when flag && !(use_t && err < t) (classify.cpp:63-66,
// 111-126); the k-th kept region (k = offsets[block] + rank in the block, the
// filter's order) becomes link[k] = j | axis << 56 and pest[k] = est[j], and
// the next k_evaluate derives children 2k, 2k+1 from that row
// (geometry.cpp:122-141, evaluate.cuh load_geometry).  No geometry moves
// here: 10-18 B read per region, 16 B written per kept region, all coalesced.
constexpr int kLinkThreads = 256;
constexpr int kLinkPer = static_cast<int>(kBlock) / kLinkThreads;  // 8 consecutive regions

// One thread's 8 consecutive regions of a 2048-block, as loaded.
struct LinkRegs {
  uint2 fw, aw;  // flag / axis bytes
  double2 xv[kLinkPer / 2], ev[kLinkPer / 2];
};

// every load issued before any use: flag / axis as 8-byte words, est / err
// as 16-byte pairs (the block start is 2048-aligned, so all are aligned)
__device__ __forceinline__ void link_load(LinkRegs& R, int64_t m, int64_t b,
                                          const uint8_t* __restrict__ flag, int use_t,
                                          const double* __restrict__ est,
                                          const double* __restrict__ err,
                                          const uint8_t* __restrict__ axis) {
  const int64_t base = b * kBlock;
  const int n = static_cast<int>(m - base < kBlock ? m - base : kBlock);
  const int i0 = threadIdx.x * kLinkPer;
  R.fw = make_uint2(0u, 0u);
  R.aw = make_uint2(0u, 0u);
  if (i0 + kLinkPer <= n) {
    R.fw = __ldg(reinterpret_cast<const uint2*>(flag + base + i0));
    R.aw = __ldg(reinterpret_cast<const uint2*>(axis + base + i0));
#pragma unroll
    for (int u = 0; u < kLinkPer / 2; ++u) {
      R.xv[u] = __ldg(reinterpret_cast<const double2*>(est + base + i0) + u);
      R.ev[u] = use_t ? __ldg(reinterpret_cast<const double2*>(err + base + i0) + u)
                      : make_double2(0.0, 0.0);
    }
  } else {  // the batch's ragged last block
    uint8_t fb[kLinkPer] = {}, ab[kLinkPer] = {};
    double xs[kLinkPer] = {}, es[kLinkPer] = {};
#pragma unroll
    for (int u = 0; u < kLinkPer; ++u)
      if (i0 + u < n) {
        fb[u] = __ldg(flag + base + i0 + u);
        ab[u] = __ldg(axis + base + i0 + u);
        xs[u] = __ldg(est + base + i0 + u);
        if (use_t) es[u] = __ldg(err + base + i0 + u);
      }
#pragma unroll
    for (int u = 0; u < kLinkPer; ++u) {
      (u < 4 ? R.fw.x : R.fw.y) |= static_cast<unsigned>(fb[u]) << (8 * (u & 3));
      (u < 4 ? R.aw.x : R.aw.y) |= static_cast<unsigned>(ab[u]) << (8 * (u & 3));
    }
#pragma unroll
    for (int u = 0; u < kLinkPer / 2; ++u) {
      R.xv[u] = make_double2(xs[2 * u], xs[2 * u + 1]);
      R.ev[u] = make_double2(es[2 * u], es[2 * u + 1]);
    }
  }
}

struct LinkSmem {
  uint64_t link[kBlock];
  double pest[kBlock];
  int warp[kLinkThreads / 32 + 1];
};

// kept = flag && !(use_t && err < t) (classify.cpp:63-66); the block's kept
// regions in order, from rank offsets[b] on.  Ends with a barrier (S reusable).
__device__ __forceinline__ void link_block(LinkSmem& S, const LinkRegs& R, int64_t b, int use_t,
                                           double t, const int64_t* __restrict__ offsets,
                                           uint64_t* __restrict__ link,
                                           double* __restrict__ pest) {
  constexpr int W = kLinkThreads / 32;
  const int64_t base = b * kBlock;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int i0 = threadIdx.x * kLinkPer;
  unsigned keep = 0;
#pragma unroll
  for (int u = 0; u < kLinkPer; ++u) {
    const unsigned f = ((u < 4 ? R.fw.x : R.fw.y) >> (8 * (u & 3))) & 0xffu;
    const double e = (u & 1) ? R.ev[u / 2].y : R.ev[u / 2].x;
    keep |= (f != 0 && !(use_t && e < t)) ? (1u << u) : 0u;
  }
  // rank of the thread's first kept region in the block: warp scan + block scan
  const int c = __popc(keep);
  int incl = c;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  if (lane == 31) S.warp[wid] = incl;
  __syncthreads();
  if (threadIdx.x == 0) {
    int run = 0;
#pragma unroll
    for (int w = 0; w < W; ++w) {
      const int v = S.warp[w];
      S.warp[w] = run;
      run += v;
    }
    S.warp[W] = run;
  }
  __syncthreads();
  int r = S.warp[wid] + incl - c;
  // stage the block's entries in rank order, then write them out coalesced
#pragma unroll
  for (int u = 0; u < kLinkPer; ++u) {
    if (!((keep >> u) & 1u)) continue;
    const unsigned ax = ((u < 4 ? R.aw.x : R.aw.y) >> (8 * (u & 3))) & 0xffu;
    S.link[r] = static_cast<uint64_t>(base + i0 + u) | (static_cast<uint64_t>(ax) << 56);
    S.pest[r] = (u & 1) ? R.xv[u / 2].y : R.xv[u / 2].x;
    ++r;
  }
  __syncthreads();
  const int total = S.warp[W];
  const int64_t k0 = offsets[b];
  for (int i = threadIdx.x; i < total; i += kLinkThreads) {
    link[k0 + i] = S.link[i];
    pest[k0 + i] = S.pest[i];
  }
  __syncthreads();
}

// One CTA per 2048-block.
__global__ void __launch_bounds__(kLinkThreads)
    k_link(int64_t m, const uint8_t* __restrict__ flag, int use_t, double t,
           const int64_t* __restrict__ offsets, const double* __restrict__ est,
           const double* __restrict__ err, const uint8_t* __restrict__ axis,
           uint64_t* __restrict__ link, double* __restrict__ pest) {
  __shared__ __align__(16) LinkSmem S;
  pdl_trigger();  // the next k_evaluate may launch (it waits for this grid in pdl_wait)
  LinkRegs R;
  link_load(R, m, blockIdx.x, flag, use_t, est, err, axis);
  link_block(S, R, blockIdx.x, use_t, t, offsets, link, pest);
}

// Persistent form: a grid of resident CTAs walks the blocks (b += gridDim.x)
// with the next block's loads in flight while the current one is ranked and
// written -- no wave tail, and the loads of block b + grid overlap block b's
// scan / stores.
__global__ void __launch_bounds__(kLinkThreads)
    k_link_p(int64_t m, int64_t nblk, const uint8_t* __restrict__ flag, int use_t, double t,
             const int64_t* __restrict__ offsets, const double* __restrict__ est,
             const double* __restrict__ err, const uint8_t* __restrict__ axis,
             uint64_t* __restrict__ link, double* __restrict__ pest) {
  __shared__ __align__(16) LinkSmem S;
  pdl_trigger();
  int64_t b = blockIdx.x;
  if (b >= nblk) return;
  LinkRegs cur, nxt;
  link_load(cur, m, b, flag, use_t, est, err, axis);
  for (; b < nblk; b += gridDim.x) {
    const int64_t bn = b + gridDim.x;
    if (bn < nblk) link_load(nxt, m, bn, flag, use_t, est, err, axis);
    link_block(S, cur, b, use_t, t, offsets, link, pest);
    cur = nxt;
  }
}

// PAGANI_LINK_PERSISTENT=1 selects k_link_p (measured slower on B200: 18.1
// vs 15.2 us for a 1233-block f1 launch, 20.2 vs 18.1 ms per bench step --
// 104 registers leave 2 CTAs per SM, and one CTA's serial scan / stage /
// store per block is the critical path, not the loads).
static bool link_persistent() {
  static const bool on = [] {
    const char* e = std::getenv("PAGANI_LINK_PERSISTENT");
    return e && std::atoi(e) != 0;
  }();
  return on;
}

void launch_link(cudaStream_t st, int64_t m, const uint8_t* flag, int use_t, double t,
                 const int64_t* offsets, const double* est, const double* err,
                 const uint8_t* axis, uint64_t* link, double* pest) {
  const int64_t nblk = nblocks_of(m);
  if (nblk == 0) return;
  if (link_persistent()) {
    static const int slots = [] {
      int d = 0, sms = 148, per = 1;
      cudaGetDevice(&d);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, d);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_link_p, kLinkThreads, 0);
      return sms * (per > 0 ? per : 1);
    }();
    const int64_t g = nblk < slots ? nblk : slots;
    k_link_p<<<static_cast<unsigned>(g), kLinkThreads, 0, st>>>(m, nblk, flag, use_t, t, offsets,
                                                                est, err, axis, link, pest);
    return;
  }
  k_link<<<static_cast<unsigned>(nblk), kLinkThreads, 0, st>>>(m, flag, use_t, t, offsets, est,
                                                               err, axis, link, pest);
}

void launch_compact(cudaStream_t st, int n, int64_t m, int64_t cap, const uint8_t* flag,
                    const int64_t* offsets, const double* low, const double* len,
                    const double* est, const double* err, const int32_t* axis,
                    const double* pest, const double* perr, double* klow, double* klen,
                    double* kest, double* kerr, int32_t* kaxis, double* kpest, double* kperr) {
  const int64_t nblk = nblocks_of(m);
  if (nblk == 0) return;
  k_compact<<<static_cast<unsigned>(nblk), kSplitThreads, 0, st>>>(
      n, m, cap, flag, offsets, low, len, est, err, axis, pest, perr, klow, klen, kest, kerr,
      kaxis, kpest, kperr);
}

void launch_refine(cudaStream_t st, int64_t m, const double* est, const double* raw,
                   const double* pest, double* out) {
  if (m > 0) k_refine<<<grid_for(m, 256), 256, 0, st>>>(m, est, raw, pest, out);
}
void launch_classify(cudaStream_t st, int64_t m, const double* est, const double* err,
                     double tau, int enabled, uint8_t* flags) {
  if (m > 0) k_classify<<<grid_for(m, 256), 256, 0, st>>>(m, est, err, tau, enabled, flags);
}
void launch_apply_threshold(cudaStream_t st, int64_t m, const double* err, double t,
                            uint8_t* flags) {
  if (m > 0) k_apply_threshold<<<grid_for(m, 256), 256, 0, st>>>(m, err, t, flags);
}
void launch_serial_volume(cudaStream_t st, int n, int64_t m, int64_t cap, const double* len,
                          const uint8_t* flag, int which, double* out) {
  k_serial_volume<<<1, 1, 0, st>>>(n, m, cap, len, flag, which, out);
}
void launch_kept_partials(cudaStream_t st, int64_t m, const uint8_t* flag, int use_t, double t,
                          const double* err, const double* est, double* part) {
  k_kept_partials<<<1, 1, 0, st>>>(m, flag, use_t, t, err, est, part);
}
void launch_math(cudaStream_t st, int which, int64_t m, const double* x, double* y) {
  if (m > 0) k_math<<<grid_for(m, 256), 256, 0, st>>>(which, m, x, y);
}

void launch_call_integrand(cudaStream_t st, int fid, int n, int64_t m, const double* x,
                           const IntegrandParams& ip, double* y) {
  if (m <= 0) return;
  const unsigned g = grid_for(m, 128);
  switch (fid) {
    case 1: k_call<F1><<<g, 128, 0, st>>>(n, m, x, ip, y); break;
    case 2: k_call<F2><<<g, 128, 0, st>>>(n, m, x, ip, y); break;
    case 3: k_call<F3><<<g, 128, 0, st>>>(n, m, x, ip, y); break;
    case 4: k_call<F4><<<g, 128, 0, st>>>(n, m, x, ip, y); break;
    case 5: k_call<F5><<<g, 128, 0, st>>>(n, m, x, ip, y); break;
    case 6: k_call<F6><<<g, 128, 0, st>>>(n, m, x, ip, y); break;
    case 7: k_call<F7><<<g, 128, 0, st>>>(n, m, x, ip, y); break;
    case 8: k_call<F8><<<g, 128, 0, st>>>(n, m, x, ip, y); break;
    case 100: k_call<TConst><<<g, 128, 0, st>>>(n, m, x, ip, y); break;
    case 101: k_call<TMonomial><<<g, 128, 0, st>>>(n, m, x, ip, y); break;
    case 102: k_call<TRough><<<g, 128, 0, st>>>(n, m, x, ip, y); break;
    case 103: k_call<TNanBox><<<g, 128, 0, st>>>(n, m, x, ip, y); break;
    case 104: k_call<TPocket><<<g, 128, 0, st>>>(n, m, x, ip, y); break;
    case 105: k_call<TCosSum><<<g, 128, 0, st>>>(n, m, x, ip, y); break;
    case 106: k_call<TExpSq><<<g, 128, 0, st>>>(n, m, x, ip, y); break;
    default: break;
  }
}

}  // namespace pgn
