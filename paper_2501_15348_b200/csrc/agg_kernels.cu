// Neighbourhood-aggregation kernels for sm_100a.
//
//   K1 agg_scratch   pull SpMM over the in-CSR          (ref src/aggregate.cpp:55-115)
//   K2 agg_delta     delta-SpMM over dst-grouped signed COO (ref src/aggregate.cpp:117-207)
//   K3 agg_backward  transposed SpMM as a pull over the out-CSR (ref src/aggregate.cpp:209-246)
//
// All three are HBM-bound gathers of feature rows. A row is owned by a group
// of G lanes (G = width / VEC rounded to a power of two, <= 32); each lane
// moves VEC contiguous floats with one vector load, so a 128-wide fp32 row is
// one fully coalesced 512 B warp access. Edge indices are fetched G at a time
// (coalesced) and broadcast by shuffle; gathers are issued UNR rows ahead of
// the in-order accumulation, so each row's reduction order is exactly the
// reference's (ascending source within a destination; deletions before
// insertions for the delta), which keeps results deterministic and makes the
// fp32 path differ from the fp64 reference only by rounding.
#include "agg_kernels.h"
#include "common.cuh"

#include <algorithm>
#include <cfloat>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

namespace dgnn {
namespace cuda {
namespace {

constexpr int kThreads = 256;
constexpr int kUnroll = 4;

template <int V>
struct VecLoad;
template <>
struct VecLoad<4> {
  __device__ static void ld(float (&r)[4], const float* p) {
    float4 x = __ldg(reinterpret_cast<const float4*>(p));
    r[0] = x.x; r[1] = x.y; r[2] = x.z; r[3] = x.w;
  }
  __device__ static void st(float* p, const float (&r)[4]) {
    *reinterpret_cast<float4*>(p) = make_float4(r[0], r[1], r[2], r[3]);
  }
  __device__ static void ld_rw(float (&r)[4], const float* p) {
    float4 x = *reinterpret_cast<const float4*>(p);
    r[0] = x.x; r[1] = x.y; r[2] = x.z; r[3] = x.w;
  }
};
template <>
struct VecLoad<2> {
  __device__ static void ld(float (&r)[2], const float* p) {
    float2 x = __ldg(reinterpret_cast<const float2*>(p));
    r[0] = x.x; r[1] = x.y;
  }
  __device__ static void st(float* p, const float (&r)[2]) {
    *reinterpret_cast<float2*>(p) = make_float2(r[0], r[1]);
  }
  __device__ static void ld_rw(float (&r)[2], const float* p) {
    float2 x = *reinterpret_cast<const float2*>(p);
    r[0] = x.x; r[1] = x.y;
  }
};
template <>
struct VecLoad<1> {
  __device__ static void ld(float (&r)[1], const float* p) { r[0] = __ldg(p); }
  __device__ static void st(float* p, const float (&r)[1]) { p[0] = r[0]; }
  __device__ static void ld_rw(float (&r)[1], const float* p) { r[0] = *p; }
};

template <int V>
__device__ inline void ld_int(int32_t (&r)[V], const int32_t* p) {
#pragma unroll
  for (int i = 0; i < V; ++i) r[i] = p[i];
}
template <int V>
__device__ inline void st_int(int32_t* p, const int32_t (&r)[V]) {
#pragma unroll
  for (int i = 0; i < V; ++i) p[i] = r[i];
}

// Per-element update of one gathered source row into the accumulator.
template <int KIND, int V>
__device__ inline void accumulate(float (&acc)[V], int32_t (&arg)[V], const float (&x)[V],
                                  int32_t u) {
#pragma unroll
  for (int i = 0; i < V; ++i) {
    if (KIND == kAggSum || KIND == kAggMean) {
      acc[i] += x[i];
    } else if (KIND == kAggMax) {
      if (arg[i] < 0 || x[i] > acc[i]) { acc[i] = x[i]; arg[i] = u; }
    } else {
      if (arg[i] < 0 || x[i] < acc[i]) { acc[i] = x[i]; arg[i] = u; }
    }
  }
}

// ---------------------------------------------------------------- K1 scratch
template <int V, int G, int KIND>
__global__ void __launch_bounds__(kThreads)
k_agg_scratch(int n, int w, int c0, int wc, const int64_t* __restrict__ ptr,
              const int32_t* __restrict__ idx, const float* __restrict__ F, float* __restrict__ out,
              float* __restrict__ degree, float* __restrict__ msum, int32_t* __restrict__ argext) {
  // columns [c0, c0 + wc) of a row-major n x w operand (L2-sized column slice)
  const int lane = threadIdx.x & 31;
  const int gl = lane & (G - 1);
  constexpr int kRowsPerWarp = 32 / G;
  const int64_t warp_global = (static_cast<int64_t>(blockIdx.x) * kThreads + threadIdx.x) >> 5;
  const int64_t warp_stride = (static_cast<int64_t>(gridDim.x) * kThreads) >> 5;
  const int nchunk = (wc + G * V - 1) / (G * V);
  const int cend = c0 + wc;
  for (int64_t vbase = warp_global * kRowsPerWarp; vbase < n; vbase += warp_stride * kRowsPerWarp) {
    const int64_t v = vbase + lane / G;
    const bool valid = v < n;
    const int64_t beg = valid ? ptr[v] : 0;
    const int deg = valid ? static_cast<int>(ptr[v + 1] - beg) : 0;
    const int maxdeg = __reduce_max_sync(0xffffffffu, deg);
    for (int k = 0; k < nchunk; ++k) {
      const int c = c0 + (k * G + gl) * V;
      const bool cact = valid && c < cend;
      float acc[V];
      int32_t arg[V];
#pragma unroll
      for (int i = 0; i < V; ++i) {
        acc[i] = KIND == kAggMax ? -INFINITY : (KIND == kAggMin ? INFINITY : 0.f);
        arg[i] = -1;
      }
      for (int eb = 0; eb < maxdeg; eb += G) {
        const int my_e = eb + gl;
        const int32_t my_u = my_e < deg ? idx[beg + my_e] : 0;
        DGNN_DCHECK(my_u >= 0 && my_u < n);
        const int cnt = min(G, maxdeg - eb);
        for (int j0 = 0; j0 < cnt; j0 += kUnroll) {
          float x[kUnroll][V];
          int32_t u[kUnroll];
#pragma unroll
          for (int q = 0; q < kUnroll; ++q) {
            u[q] = __shfl_sync(0xffffffffu, my_u, (j0 + q) & (G - 1), G);
            if (cact && j0 + q < cnt && eb + j0 + q < deg) {
              VecLoad<V>::ld(x[q], F + static_cast<int64_t>(u[q]) * w + c);
            }
          }
#pragma unroll
          for (int q = 0; q < kUnroll; ++q) {
            if (cact && j0 + q < cnt && eb + j0 + q < deg) accumulate<KIND, V>(acc, arg, x[q], u[q]);
          }
        }
      }
      if (cact) {
        float* o = out + v * w + c;
        if (KIND == kAggMean) {
          VecLoad<V>::st(msum + v * w + c, acc);
          float r[V];
          const float dg = static_cast<float>(deg);
#pragma unroll
          for (int i = 0; i < V; ++i) r[i] = deg > 0 ? acc[i] / dg : 0.f;
          VecLoad<V>::st(o, r);
          if (c == 0) degree[v] = dg;
        } else {
          VecLoad<V>::st(o, acc);
          if (KIND == kAggMax || KIND == kAggMin) st_int<V>(argext + v * w + c, arg);
        }
      }
    }
  }
}

// ---------------------------------------------------------------- K2 delta
// rows[r] = destination, entries ent[row_ptr[r] .. row_ptr[r+1]) = deletions
// (encoded ~src, ascending src) followed by insertions (src, ascending).
template <int V, int G, int KIND>
__global__ void __launch_bounds__(kThreads)
k_agg_delta(int n_rows, int w, const int32_t* __restrict__ rows, const int32_t* __restrict__ row_ptr,
            const int32_t* __restrict__ ent, const float* __restrict__ Fp, const float* __restrict__ Fc,
            float* __restrict__ values, float* __restrict__ degree, float* __restrict__ msum,
            int32_t* __restrict__ argext) {
  const int lane = threadIdx.x & 31;
  const int gl = lane & (G - 1);
  constexpr int kRowsPerWarp = 32 / G;
  const int64_t warp_global = (static_cast<int64_t>(blockIdx.x) * kThreads + threadIdx.x) >> 5;
  const int64_t warp_stride = (static_cast<int64_t>(gridDim.x) * kThreads) >> 5;
  const int nchunk = (w + G * V - 1) / (G * V);
  for (int64_t rbase = warp_global * kRowsPerWarp; rbase < n_rows; rbase += warp_stride * kRowsPerWarp) {
    const int64_t r = rbase + lane / G;
    const bool valid = r < n_rows;
    const int64_t v = valid ? rows[r] : 0;
    const int beg = valid ? row_ptr[r] : 0;
    const int cnt_row = valid ? row_ptr[r + 1] - beg : 0;
    const int maxcnt = __reduce_max_sync(0xffffffffu, cnt_row);
    int dnet = 0;  // insertions - deletions (mean degree update)
    for (int k = 0; k < nchunk; ++k) {
      const int c = (k * G + gl) * V;
      const bool cact = valid && c < w;
      float acc[V];
      int32_t arg[V];
      float* accp = (KIND == kAggMean ? msum : values) + v * w + c;
      if (cact) {
        VecLoad<V>::ld_rw(acc, accp);
        if (KIND == kAggMax || KIND == kAggMin) ld_int<V>(arg, argext + v * w + c);
      }
      for (int eb = 0; eb < maxcnt; eb += G) {
        const int my_e = eb + gl;
        const int32_t my_s = my_e < cnt_row ? ent[beg + my_e] : 0;
        const int cnt = min(G, maxcnt - eb);
        for (int j0 = 0; j0 < cnt; j0 += kUnroll) {
          float x[kUnroll][V];
          int32_t s[kUnroll];
#pragma unroll
          for (int q = 0; q < kUnroll; ++q) {
            s[q] = __shfl_sync(0xffffffffu, my_s, (j0 + q) & (G - 1), G);
            const bool live = cact && j0 + q < cnt && eb + j0 + q < cnt_row;
            if (live) {
              if (s[q] < 0) {
                if (KIND == kAggSum || KIND == kAggMean)
                  VecLoad<V>::ld(x[q], Fp + static_cast<int64_t>(~s[q]) * w + c);
              } else {
                VecLoad<V>::ld(x[q], Fc + static_cast<int64_t>(s[q]) * w + c);
              }
            }
          }
#pragma unroll
          for (int q = 0; q < kUnroll; ++q) {
            const bool live = cact && j0 + q < cnt && eb + j0 + q < cnt_row;
            if (!live) continue;
            if (KIND == kAggSum || KIND == kAggMean) {
              if (s[q] < 0) {
#pragma unroll
                for (int i = 0; i < V; ++i) acc[i] -= x[q][i];
              } else {
#pragma unroll
                for (int i = 0; i < V; ++i) acc[i] += x[q][i];
              }
              if (k == 0) dnet += s[q] < 0 ? -1 : 1;
            } else if (s[q] >= 0) {
              accumulate<KIND, V>(acc, arg, x[q], s[q]);  // max/min: insert-only
            }
          }
        }
      }
      if (cact) {
        VecLoad<V>::st(accp, acc);
        if (KIND == kAggMax || KIND == kAggMin) st_int<V>(argext + v * w + c, arg);
      }
    }
    if (KIND == kAggMean) {
      // Renormalise the touched row (ref src/aggregate.cpp:195-205).
      const float dg = valid ? degree[v] + static_cast<float>(dnet) : 0.f;
      const bool keep = dg > 1e-12f;
      for (int k = 0; k < nchunk; ++k) {
        const int c = (k * G + gl) * V;
        if (!(valid && c < w)) continue;
        float ms[V], r[V];
        VecLoad<V>::ld_rw(ms, msum + v * w + c);
#pragma unroll
        for (int i = 0; i < V; ++i) {
          r[i] = keep ? ms[i] / dg : 0.f;
          if (!keep) ms[i] = 0.f;
        }
        VecLoad<V>::st(values + v * w + c, r);
        if (!keep) VecLoad<V>::st(msum + v * w + c, ms);
      }
      __syncwarp();
      if (valid && gl == 0) degree[v] = keep ? dg : 0.f;
    }
  }
}

// L2 eviction-priority policies for the delta gathers: the compact
// changed-row block is re-read ~20x (every out-edge of a changed node appears
// in G- and G+) and is kept (evict_last); destination rows and structural
// source rows are touched once (evict_first).
__device__ __forceinline__ uint64_t l2_policy_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t l2_policy_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ float4 ld_nc_hint(const float* p, uint64_t pol) {
  float4 r;
  asm volatile("ld.global.nc.L2::cache_hint.v4.f32 {%0, %1, %2, %3}, [%4], %5;"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
               : "l"(p), "l"(pol));
  return r;
}
__device__ __forceinline__ void st_hint(float* p, float4 v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v4.f32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(p), "f"(v.x),
               "f"(v.y), "f"(v.z), "f"(v.w), "l"(pol)
               : "memory");
}
__device__ __forceinline__ float4 ld_hint(const float* p, uint64_t pol) {
  float4 r;
  asm volatile("ld.global.L2::cache_hint.v4.f32 {%0, %1, %2, %3}, [%4], %5;"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
               : "l"(p), "l"(pol));
  return r;
}

// K2, pipelined (sum / mean, w <= 128 * U / ..., 16 B-aligned rows). One
// destination row per group of G lanes, each lane owning U consecutive
// float4s (4U columns), so 32 / G rows are in flight per warp step (U = 2
// doubles the rows in flight at w = 64 / 128 over one float4 per lane).
// The dependent index chain (row meta -> entries -> source rows) is software
// pipelined across steps: each step issues the row metadata two steps ahead
// and the first G entries one step ahead together with this step's
// destination-row and source-row loads, so a step costs one memory round trip
// instead of three. Entries are applied in the reference's order (deletions,
// then insertions, ascending source); with the compact block a persisting
// changed-source pair is one entry (its difference row) at the deletion's place.
template <int G, int U, bool MEAN, int MINB = 1, bool STRUCT = false, int KU = kUnroll>
__global__ void __launch_bounds__(kThreads, MINB)
k_agg_delta_v4(int n_rows, int w, int32_t num_nodes, const int32_t* __restrict__ rows,
               const int32_t* __restrict__ row_ptr, const int32_t* __restrict__ ent,
               const float* __restrict__ Fp, const float* __restrict__ Fc,
               const float* __restrict__ Cp, const float* __restrict__ Cc,
               float* __restrict__ values, float* __restrict__ degree, float* __restrict__ msum,
               int st_evict_first, const int32_t* __restrict__ changed) {
  // STRUCT: structural mode (Fp == Fc = one matrix H, no compact
  // block): folded pairs ~(N + p) cancel and are skipped, insertions N + p
  // read H[changed[p]] — Agg_{G_t}(H) from Agg_{G_{t-1}}(H)
  constexpr int R = 32 / G;
  const int lane = threadIdx.x & 31, gl = lane & (G - 1), sub = lane / G;
  const int64_t wg = (static_cast<int64_t>(blockIdx.x) * kThreads + threadIdx.x) >> 5;
  const int64_t step = ((static_cast<int64_t>(gridDim.x) * kThreads) >> 5) * R;
  // float4 u of a lane covers columns (u * G + gl) * 4: each load instruction
  // of a G-lane group reads one contiguous 16G-byte segment of the row
  const int c = gl * 4;
  const bool cact = c < w;
  auto col_ok = [&](int u) { return c + 4 * G * u < w; };
  const uint64_t keep = l2_policy_last(), once = l2_policy_first();
  struct Meta {
    int32_t v, beg, cnt;
  };
  auto meta = [&](int64_t rb) {
    Meta m{0, 0, 0};
    const int64_t r = rb + sub;
    if (r < n_rows) {
      m.v = rows[r];
      m.beg = row_ptr[r];
      m.cnt = row_ptr[r + 1] - m.beg;
      DGNN_DCHECK(m.v >= 0 && m.cnt >= 0);
    }
    return m;
  };
  auto first_ent = [&](const Meta& m) { return gl < m.cnt ? ent[m.beg + gl] : 0; };
  int64_t rb = wg * R;
  Meta m0 = meta(rb), m1 = meta(rb + step);
  int32_t e0 = first_ent(m0);
  float d0 = MEAN && rb + sub < n_rows ? degree[m0.v] : 0.f;
  for (; rb < n_rows; rb += step) {
    const Meta m2 = meta(rb + 2 * step);
    const int32_t e1 = first_ent(m1);
    const float d1 = MEAN && rb + step + sub < n_rows ? degree[m1.v] : 0.f;
    const bool valid = rb + sub < n_rows;
    float* accp = (MEAN ? msum : values) + static_cast<int64_t>(m0.v) * w + c;
    float4 acc[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      acc[u] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (valid && col_ok(u)) acc[u] = ld_hint(accp + 4 * G * u, once);
    }
    const int maxcnt = __reduce_max_sync(0xffffffffu, m0.cnt);
    int dnet = 0;
    for (int eb = 0; eb < maxcnt; eb += G) {
      const int32_t my_s = eb == 0 ? e0 : (eb + gl < m0.cnt ? ent[m0.beg + eb + gl] : 0);
      const int cnt = min(G, maxcnt - eb);
      for (int j0 = 0; j0 < cnt; j0 += KU) {
        float4 x[KU][U];
        int32_t s[KU];
#pragma unroll
        for (int q = 0; q < KU; ++q) {
          s[q] = __shfl_sync(0xffffffffu, my_s, (j0 + q) & (G - 1), G);
          if (valid && cact && j0 + q < cnt && eb + j0 + q < m0.cnt &&
              !(STRUCT && s[q] < 0 && ~s[q] >= num_nodes)) {
            const int32_t u0 = s[q] < 0 ? ~s[q] : s[q];
            const bool cpt = u0 >= num_nodes;
            const float* src;
            if (STRUCT && cpt) src = Fc + static_cast<int64_t>(changed[u0 - num_nodes]) * w + c;
            else if (cpt) src = (s[q] < 0 ? Cp : Cc) + static_cast<int64_t>(u0 - num_nodes) * w + c;
            else src = (s[q] < 0 ? Fp : Fc) + static_cast<int64_t>(u0) * w + c;
#pragma unroll
            for (int u = 0; u < U; ++u)
              if (col_ok(u)) x[q][u] = ld_nc_hint(src + 4 * G * u, cpt && !STRUCT ? keep : once);
          }
        }
#pragma unroll
        for (int q = 0; q < KU; ++q) {
          if (!(valid && j0 + q < cnt && eb + j0 + q < m0.cnt)) continue;
          if (STRUCT && s[q] < 0 && ~s[q] >= num_nodes) continue;  // persisting pair: cancels
          // a compact-block deletion is a folded (deletion, insertion) pair
          if (MEAN) dnet += s[q] >= 0 ? 1 : (~s[q] >= num_nodes ? 0 : -1);
          if (!cact) continue;
#pragma unroll
          for (int u = 0; u < U; ++u) {
            if (!col_ok(u)) continue;
            if (s[q] < 0) {
              acc[u].x -= x[q][u].x; acc[u].y -= x[q][u].y; acc[u].z -= x[q][u].z; acc[u].w -= x[q][u].w;
            } else {
              acc[u].x += x[q][u].x; acc[u].y += x[q][u].y; acc[u].z += x[q][u].z; acc[u].w += x[q][u].w;
            }
          }
        }
      }
    }
    if (valid && cact) {
      if (MEAN) {
        // renormalise the touched row (ref src/aggregate.cpp:195-205)
        const float dg = d0 + static_cast<float>(dnet);
        const bool live = dg > 1e-12f;
        float* vp = values + static_cast<int64_t>(m0.v) * w + c;
#pragma unroll
        for (int u = 0; u < U; ++u) {
          if (!col_ok(u)) continue;
          const float4 ms = live ? acc[u] : make_float4(0.f, 0.f, 0.f, 0.f);
          *reinterpret_cast<float4*>(accp + 4 * G * u) = ms;
          *reinterpret_cast<float4*>(vp + 4 * G * u) =
              live ? make_float4(acc[u].x / dg, acc[u].y / dg, acc[u].z / dg, acc[u].w / dg) : ms;
        }
        if (gl == 0) degree[m0.v] = live ? dg : 0.f;
      } else {
#pragma unroll
        for (int u = 0; u < U; ++u) {
          if (!col_ok(u)) continue;
          if (st_evict_first) st_hint(accp + 4 * G * u, acc[u], once);
          else *reinterpret_cast<float4*>(accp + 4 * G * u) = acc[u];
        }
      }
    }
    m0 = m1;
    m1 = m2;
    e0 = e1;
    d0 = d1;
  }
}

// K1 / K3 for sum (the configs' aggregation): out[v] = (addend[v]) + sum over
// the CSR row of F[u], ascending u. G lanes per row with U float4s each, so
// 32 / G rows are gathered concurrently per warp (more independent 16 B
// gathers in flight than one float4 per lane), and the next G indices of a
// row are loaded before the current batch's gathers are consumed.
template <int G, int U>
__global__ void __launch_bounds__(kThreads)
k_spmm_sum(int n, int w, const int64_t* __restrict__ ptr, const int32_t* __restrict__ idx,
           const float* __restrict__ F, float* out, const float* addend) {
  constexpr int R = 32 / G;
  const int lane = threadIdx.x & 31, gl = lane & (G - 1), sub = lane / G;
  const int64_t warp_global = (static_cast<int64_t>(blockIdx.x) * kThreads + threadIdx.x) >> 5;
  const int64_t warp_stride = (static_cast<int64_t>(gridDim.x) * kThreads) >> 5;
  // float4 u of a lane covers columns (u * G + gl) * 4 (coalesced 16G-byte
  // segments per load instruction)
  const int c = gl * 4;
  const bool cin = c < w;
  auto col_ok = [&](int u) { return c + 4 * G * u < w; };
  for (int64_t vbase = warp_global * R; vbase < n; vbase += warp_stride * R) {
    const int64_t v = vbase + sub;
    const bool valid = v < n;
    const int64_t beg = valid ? ptr[v] : 0;
    const int deg = valid ? static_cast<int>(ptr[v + 1] - beg) : 0;
    const int maxdeg = __reduce_max_sync(0xffffffffu, deg);
    const bool cact = valid && cin;
    float4 acc[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      acc[u] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (addend != nullptr && cact && col_ok(u))
        acc[u] = *reinterpret_cast<const float4*>(addend + v * w + c + 4 * G * u);
    }
    int32_t my_u = gl < deg ? idx[beg + gl] : 0;
    DGNN_DCHECK(my_u >= 0 && my_u < n);
    for (int eb = 0; eb < maxdeg; eb += G) {
      // next batch's indices in flight with this batch's gathers
      const int32_t nxt_u = eb + G + gl < deg ? idx[beg + eb + G + gl] : 0;
      DGNN_DCHECK(nxt_u >= 0 && nxt_u < n);
      const int cnt = min(G, maxdeg - eb);
      for (int j0 = 0; j0 < cnt; j0 += kUnroll) {
        float4 x[kUnroll][U];
#pragma unroll
        for (int q = 0; q < kUnroll; ++q) {
          const int32_t uu = __shfl_sync(0xffffffffu, my_u, (j0 + q) & (G - 1), G);
          if (cact && j0 + q < cnt && eb + j0 + q < deg) {
            const float* src = F + static_cast<int64_t>(uu) * w + c;
#pragma unroll
            for (int u = 0; u < U; ++u)
              if (col_ok(u)) x[q][u] = __ldg(reinterpret_cast<const float4*>(src + 4 * G * u));
          }
        }
#pragma unroll
        for (int q = 0; q < kUnroll; ++q) {
          if (!(cact && j0 + q < cnt && eb + j0 + q < deg)) continue;
#pragma unroll
          for (int u = 0; u < U; ++u) {
            if (!col_ok(u)) continue;
            acc[u].x += x[q][u].x; acc[u].y += x[q][u].y; acc[u].z += x[q][u].z; acc[u].w += x[q][u].w;
          }
        }
      }
      my_u = nxt_u;
    }
    if (cact) {
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (col_ok(u)) *reinterpret_cast<float4*>(out + v * w + c + 4 * G * u) = acc[u];
    }
  }
}

// U float4s per lane for k_spmm_sum (0: not applicable); DGNN_SPMM_U overrides
int spmm_u(int w) {
  static const int env = [] {
    const char* e = std::getenv("DGNN_SPMM_U");
    return e ? std::atoi(e) : -1;
  }();
  if (env == 0 || w % 4 != 0) return 0;
  int u = w % 16 == 0 && w >= 64 ? 4 : (w % 8 == 0 && w >= 32 ? 2 : 1);
  if (env > 0) u = std::min(u, env);
  return u;
}

// Deleted-contributor test for max/min (ref src/aggregate.cpp:145-153).
__global__ void k_deleted_contributor(int64_t n_del, int w, const uint64_t* __restrict__ del_keys,
                                      const int32_t* __restrict__ argext, int32_t* flag) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n_del * w;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t e = i / w;
    const int d = static_cast<int>(i - e * w);
    const int32_t src = static_cast<int32_t>(del_keys[e] >> 32);
    const int64_t dst = static_cast<int64_t>(del_keys[e] & 0xffffffffu);
    if (argext[dst * w + d] == src) atomicOr(flag, 1);
  }
}

// ---------------------------------------------------------------- K3 backward
// grad[u] = sum_{v in out(u), ascending} s_v * up[v]; s_v = 1 (sum), 1/deg(v) (mean).
// EXT (max / min): element (v, c) contributes only where argext[v][c] == u —
// the reference's scatter to the recorded contributor (ref src/aggregate.cpp:
// 234-243, v ascending) restated as a pull, so the sum order per element is
// the reference's and the result is deterministic (no atomics).
template <int V, int G, bool MEAN, bool EXT = false>
__global__ void __launch_bounds__(kThreads)
k_agg_backward(int n, int w, int c0, int wc, const int64_t* __restrict__ ptr,
               const int32_t* __restrict__ idx, const float* __restrict__ up,
               const float* __restrict__ degree, float* grad, const float* addend,
               const int32_t* __restrict__ argext = nullptr) {
  const int lane = threadIdx.x & 31;
  const int gl = lane & (G - 1);
  constexpr int kRowsPerWarp = 32 / G;
  const int64_t warp_global = (static_cast<int64_t>(blockIdx.x) * kThreads + threadIdx.x) >> 5;
  const int64_t warp_stride = (static_cast<int64_t>(gridDim.x) * kThreads) >> 5;
  const int nchunk = (wc + G * V - 1) / (G * V);
  const int cend = c0 + wc;
  for (int64_t ubase = warp_global * kRowsPerWarp; ubase < n; ubase += warp_stride * kRowsPerWarp) {
    const int64_t u = ubase + lane / G;
    const bool valid = u < n;
    const int64_t beg = valid ? ptr[u] : 0;
    const int deg = valid ? static_cast<int>(ptr[u + 1] - beg) : 0;
    const int maxdeg = __reduce_max_sync(0xffffffffu, deg);
    for (int k = 0; k < nchunk; ++k) {
      const int c = c0 + (k * G + gl) * V;
      const bool cact = valid && c < cend;
      float acc[V];
      if (addend != nullptr && cact) {  // addend may alias grad: same element, same thread
        VecLoad<V>::ld_rw(acc, addend + u * w + c);
      } else {
#pragma unroll
        for (int i = 0; i < V; ++i) acc[i] = 0.f;
      }
      for (int eb = 0; eb < maxdeg; eb += G) {
        const int my_e = eb + gl;
        const int32_t my_v = my_e < deg ? idx[beg + my_e] : 0;
        DGNN_DCHECK(my_v >= 0 && my_v < n);
        float my_s = 1.f;
        if (MEAN && my_e < deg) my_s = 1.f / degree[my_v];
        const int cnt = min(G, maxdeg - eb);
        for (int j0 = 0; j0 < cnt; j0 += kUnroll) {
          float x[kUnroll][V];
          float sc[kUnroll];
#pragma unroll
          for (int q = 0; q < kUnroll; ++q) {
            const int32_t vv = __shfl_sync(0xffffffffu, my_v, (j0 + q) & (G - 1), G);
            sc[q] = MEAN ? __shfl_sync(0xffffffffu, my_s, (j0 + q) & (G - 1), G) : 1.f;
            if (cact && j0 + q < cnt && eb + j0 + q < deg) {
              VecLoad<V>::ld(x[q], up + static_cast<int64_t>(vv) * w + c);
              if (EXT) {
                float a[V];
                VecLoad<V>::ld(a, reinterpret_cast<const float*>(argext + static_cast<int64_t>(vv) * w + c));
#pragma unroll
                for (int i = 0; i < V; ++i)
                  if (__float_as_int(a[i]) != static_cast<int32_t>(u)) x[q][i] = 0.f;
              }
            }
          }
#pragma unroll
          for (int q = 0; q < kUnroll; ++q) {
            if (cact && j0 + q < cnt && eb + j0 + q < deg) {
#pragma unroll
              for (int i = 0; i < V; ++i) {
                if (EXT) {
                  if (__float_as_int(x[q][i]) != 0) acc[i] += x[q][i];  // skip non-contributors exactly
                } else {
                  acc[i] += MEAN ? sc[q] * x[q][i] : x[q][i];
                }
              }
            }
          }
        }
      }
      if (cact) VecLoad<V>::st(grad + u * w + c, acc);
    }
  }
}


__global__ void k_mask_empty(int64_t total, int w, const int32_t* __restrict__ argext,
                             const float* __restrict__ in, float* __restrict__ out) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t v = i / w;
    out[i] = argext[v * w] < 0 ? 0.f : in[i];
  }
}

// ------------------------------------------------------------ dispatch
int pick_vec(int w, const void* a, const void* b) {
  auto al = [](const void* p, int bytes) {
    return p == nullptr || (reinterpret_cast<uintptr_t>(p) % bytes) == 0;
  };
  if (w % 4 == 0 && al(a, 16) && al(b, 16)) return 4;
  if (w % 2 == 0 && al(a, 8) && al(b, 8)) return 2;
  return 1;
}

int pick_group(int w, int vec) {
  int need = (w + vec - 1) / vec;
  int g = 1;
  while (g < need && g < 32) g <<= 1;
  return g;
}

#define DGNN_DISPATCH_G(G_RUNTIME, ...)        \
  switch (G_RUNTIME) {                         \
    case 1: { constexpr int G = 1; __VA_ARGS__; } break;   \
    case 2: { constexpr int G = 2; __VA_ARGS__; } break;   \
    case 4: { constexpr int G = 4; __VA_ARGS__; } break;   \
    case 8: { constexpr int G = 8; __VA_ARGS__; } break;   \
    case 16: { constexpr int G = 16; __VA_ARGS__; } break; \
    default: { constexpr int G = 32; __VA_ARGS__; } break; \
  }

#define DGNN_DISPATCH_V(V_RUNTIME, ...)                    \
  switch (V_RUNTIME) {                                     \
    case 4: { constexpr int V = 4; __VA_ARGS__; } break;   \
    case 2: { constexpr int V = 2; __VA_ARGS__; } break;   \
    default: { constexpr int V = 1; __VA_ARGS__; } break;  \
  }

#define DGNN_DISPATCH_KIND(K_RUNTIME, ...)                             \
  switch (K_RUNTIME) {                                                 \
    case kAggSum: { constexpr int KIND = kAggSum; __VA_ARGS__; } break;   \
    case kAggMean: { constexpr int KIND = kAggMean; __VA_ARGS__; } break; \
    case kAggMax: { constexpr int KIND = kAggMax; __VA_ARGS__; } break;   \
    default: { constexpr int KIND = kAggMin; __VA_ARGS__; } break;        \
  }

// Column-slice width for the pull SpMMs: the gathered operand's slice
// (n x wc fp32) is kept at or below an L2-resident budget so the ~E/N
// re-gathers of every source row hit L2 instead of HBM; each slice re-reads
// the index stream once. DGNN_SPMM_SLICES forces the slice count.
// the SpMM slicing experiments are opt-in by environment (read once)
bool spmm_slicing_requested() {
  static const bool on = std::getenv("DGNN_SPMM_L2_MB") != nullptr || std::getenv("DGNN_SPMM_SLICES") != nullptr;
  return on;
}

int spmm_slice_width(int n, int w, int vec) {
  static const int forced = [] {
    const char* e = std::getenv("DGNN_SPMM_SLICES");
    return e ? std::atoi(e) : 0;
  }();
  static const double budget = [] {
    const char* e = std::getenv("DGNN_SPMM_L2_MB");
    return (e ? std::atof(e) : 48.0) * 1048576.0;
  }();
  if (forced > 0 && w % forced == 0 && (w / forced) % vec == 0) return w / forced;
  // Measured on B200 at C3 (1M x 64, 20M edges): 1 slice 0.84 ms, 2: 0.89,
  // 4: 1.04, 8: 2.07 — full-row 256 B gathers beat L2-resident 32-64 B ones,
  // so slicing is off unless an explicit L2 budget is requested.
  if (!spmm_slicing_requested()) return w;
  int wc = w;
  while (static_cast<double>(n) * wc * 4.0 > budget && wc % (2 * vec) == 0 && wc / 2 >= 8) wc /= 2;
  return wc;
}

int rows_grid(int64_t rows, int g);

void launch_spmm_sum(int U, int n, int w, const int64_t* ptr, const int32_t* idx, const float* F,
                     float* out, const float* addend, cudaStream_t stream) {
  const int g = pick_group(w, 4 * U);
  const int grid = rows_grid(n, g);
  switch (U) {
    case 4:
      DGNN_DISPATCH_G(g, DGNN_LAUNCH((k_spmm_sum<G, 4>), grid, kThreads, 0, stream, n, w, ptr, idx, F, out,
                                     addend));
      break;
    case 2:
      DGNN_DISPATCH_G(g, DGNN_LAUNCH((k_spmm_sum<G, 2>), grid, kThreads, 0, stream, n, w, ptr, idx, F, out,
                                     addend));
      break;
    default:
      DGNN_DISPATCH_G(g, DGNN_LAUNCH((k_spmm_sum<G, 1>), grid, kThreads, 0, stream, n, w, ptr, idx, F, out,
                                     addend));
  }
}

int rows_grid(int64_t rows, int g) {
  const int64_t rows_per_block = (kThreads / 32) * (32 / g);
  return wave_grid(rows * kThreads / rows_per_block, kThreads, 8);
}

}  // namespace

void agg_scratch(int kind, int n, int w, const int64_t* in_ptr, const int32_t* in_src,
                 const float* feats, float* values, float* degree, float* mean_sums,
                 int32_t* argext, cudaStream_t stream) {
  if (n <= 0 || w <= 0) return;
  const int vec = pick_vec(w, feats, values);
  if (kind == kAggSum && vec == 4 && !spmm_slicing_requested()) {
    if (const int U = spmm_u(w)) {
      launch_spmm_sum(U, n, w, in_ptr, in_src, feats, values, nullptr, stream);
      return;
    }
  }
  const int wc = spmm_slice_width(n, w, vec);
  const int g = pick_group(wc, vec);
  const int grid = rows_grid(n, g);
  for (int c0 = 0; c0 < w; c0 += wc) {
    DGNN_DISPATCH_KIND(kind, DGNN_DISPATCH_V(vec, DGNN_DISPATCH_G(g,
        DGNN_LAUNCH((k_agg_scratch<V, G, KIND>), grid, kThreads, 0, stream, n, w, c0, wc, in_ptr,
                    in_src, feats, values, degree, mean_sums, argext))));
  }
}

void agg_delta(int kind, int n_rows, int w, const int32_t* rows, const int32_t* row_ptr,
               const int32_t* ent, const float* f_prev, const float* f_curr, float* values,
               float* degree, float* mean_sums, int32_t* argext, cudaStream_t stream,
               const int32_t* ent_c, int32_t num_nodes, int64_t n_changed, const float* compact,
               const int32_t* row_ptr_c) {
  if (n_rows <= 0 || w <= 0) return;
  const int vec = pick_vec(w, f_prev, values);
  const bool aligned = pick_vec(w, f_curr, mean_sums) == 4 && pick_vec(w, compact, nullptr) == 4;
  static const bool pipe_off = [] {
    const char* e = std::getenv("DGNN_DELTA_PIPE");
    return e && e[0] == '0';
  }();
  // Optional L2 set-aside for evict_last lines (the compact changed-row
  // block); DGNN_L2_PERSIST_MB, capped at the device maximum.
  static const bool l2_once = [] {
    const char* e = std::getenv("DGNN_L2_PERSIST_MB");
    if (!e) return false;
    int dev = 0, mx = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&mx, cudaDevAttrMaxPersistingL2CacheSize, dev);
    const size_t want = std::min<size_t>(static_cast<size_t>(std::atof(e) * 1048576.0), static_cast<size_t>(mx));
    cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, want);
    std::fprintf(stderr, "[dgnn] L2 persisting limit %zu bytes (device max %d)\n", want, mx);
    return true;
  }();
  (void)l2_once;
  if (ent_c == nullptr) {  // no compact block: every source is a full-matrix row
    ent_c = ent;
    row_ptr_c = row_ptr;
    num_nodes = INT32_MAX;
  }
  static const int u_env = [] {
    const char* e = std::getenv("DGNN_DELTA_U");
    return e ? std::atoi(e) : 0;
  }();
  // float4s per lane: more rows per warp step = more independent gathers in
  // flight (C4 delta, 4.8M entries: U=1 0.85 ms, U=2 0.80, U=4 0.77)
  int U = w % 8 == 0 && w >= 32 ? 2 : 1;
  if (w % 16 == 0 && w >= 64) U = 4;
  if (u_env == 1 || u_env == 2) U = std::min(U, u_env);
  if (!pipe_off && (kind == kAggSum || kind == kAggMean) && vec == 4 && aligned && w <= 128 * U) {
    const int g = pick_group(w, 4 * U);
    // DGNN_DELTA_GRID: CTAs per SM of the grid-stride launch (experiments)
    static const int per_sm = [] {
      const char* e = std::getenv("DGNN_DELTA_GRID");
      return e ? std::atoi(e) : 0;
    }();
    const int grid = per_sm > 0 ? cuda::wave_grid(static_cast<int64_t>(n_rows) * kThreads / ((kThreads / 32) * (32 / g)),
                                                  kThreads, per_sm)
                                : rows_grid(n_rows, g);
    const float* cp = compact;
    const float* cc = compact ? compact + n_changed * w : nullptr;
#define DGNN_DELTA_LAUNCH(UU, MM)                                                                    \
  DGNN_DISPATCH_G(g, DGNN_LAUNCH((k_agg_delta_v4<G, UU, MM>), grid, kThreads, 0, stream, n_rows, w, \
                                 num_nodes, rows, row_ptr_c, ent_c, f_prev, f_curr, cp, cc, values, \
                                 degree, mean_sums, st_ef, nullptr))
    // destination rows are written once per delta: evict_first keeps them
    // from displacing the compact block (DGNN_DELTA_ST_HINT=0 disables)
    static const int st_ef = [] {
      const char* e = std::getenv("DGNN_DELTA_ST_HINT");
      return e ? std::atoi(e) : 1;
    }();
    static const int minb = [] {
      const char* e = std::getenv("DGNN_DELTA_MINB");
      return e ? std::atoi(e) : 0;
    }();
    if (U == 4 && kind == kAggMean) {
      DGNN_DELTA_LAUNCH(4, true);
    } else if (U == 4 && minb == 3) {
      DGNN_DISPATCH_G(g, DGNN_LAUNCH((k_agg_delta_v4<G, 4, false, 3>), grid, kThreads, 0, stream, n_rows,
                                     w, num_nodes, rows, row_ptr_c, ent_c, f_prev, f_curr, cp, cc,
                                     values, degree, mean_sums, st_ef, nullptr))
    } else if (U == 4 && minb == 4) {
      DGNN_DISPATCH_G(g, DGNN_LAUNCH((k_agg_delta_v4<G, 4, false, 4>), grid, kThreads, 0, stream, n_rows,
                                     w, num_nodes, rows, row_ptr_c, ent_c, f_prev, f_curr, cp, cc,
                                     values, degree, mean_sums, st_ef, nullptr))
    } else if (U == 4) {
      DGNN_DELTA_LAUNCH(4, false);
    } else if (U == 2 && kind == kAggMean) {
      DGNN_DELTA_LAUNCH(2, true);
    } else if (U == 2) {
      DGNN_DELTA_LAUNCH(2, false);
    } else if (kind == kAggMean) {
      DGNN_DELTA_LAUNCH(1, true);
    } else {
      DGNN_DELTA_LAUNCH(1, false);
    }
#undef DGNN_DELTA_LAUNCH
    return;
  }
  const int g = pick_group(w, vec);
  const int grid = rows_grid(n_rows, g);
  DGNN_DISPATCH_KIND(kind, DGNN_DISPATCH_V(vec, DGNN_DISPATCH_G(g,
      DGNN_LAUNCH((k_agg_delta<V, G, KIND>), grid, kThreads, 0, stream, n_rows, w, rows, row_ptr,
                  ent, f_prev, f_curr, values, degree, mean_sums, argext))));
}

namespace {
int struct_unroll(int w) {
  int U = w % 8 == 0 && w >= 32 ? 2 : 1;
  if (w % 16 == 0 && w >= 64) U = 4;
  return U;
}
}  // namespace

bool agg_delta_struct_supported(int kind, int w, const float* h) {
  if (kind != kAggSum && kind != kAggMean) return false;
  // outputs are fresh pool blocks (256 B aligned): only h's alignment varies
  if (pick_vec(w, h, nullptr) != 4) return false;
  return w <= 128 * struct_unroll(w);
}

bool agg_delta_struct(int kind, int n_rows, int w, const int32_t* rows, const int32_t* row_ptr_c,
                      const int32_t* ent_c, int32_t num_nodes, const int32_t* changed,
                      const float* h, float* values, float* degree, float* mean_sums,
                      cudaStream_t stream) {
  if (kind != kAggSum && kind != kAggMean) return false;
  if (pick_vec(w, h, values) != 4 || pick_vec(w, mean_sums, nullptr) != 4) return false;
  const int U = struct_unroll(w);
  if (w > 128 * U) return false;
  if (n_rows <= 0) return true;
  const int g = pick_group(w, 4 * U);
  const int grid = rows_grid(n_rows, g);
#define DGNN_STRUCT_LAUNCH(UU, MM)                                                                    \
  DGNN_DISPATCH_G(g, DGNN_LAUNCH((k_agg_delta_v4<G, UU, MM, 1, true>), grid, kThreads, 0, stream,  \
                                 n_rows, w, num_nodes, rows, row_ptr_c, ent_c, h, h, nullptr,       \
                                 nullptr, values,                                                   \
                                 degree, mean_sums, 1, changed))
  const bool mean = kind == kAggMean;
  if (U == 4) {
    if (mean) DGNN_STRUCT_LAUNCH(4, true) else DGNN_STRUCT_LAUNCH(4, false)
  } else if (U == 2) {
    if (mean) DGNN_STRUCT_LAUNCH(2, true) else DGNN_STRUCT_LAUNCH(2, false)
  } else {
    if (mean) DGNN_STRUCT_LAUNCH(1, true) else DGNN_STRUCT_LAUNCH(1, false)
  }
#undef DGNN_STRUCT_LAUNCH
  return true;
}

void agg_deleted_contributor(int64_t n_del, int w, const uint64_t* del_keys,
                             const int32_t* argext, int32_t* flag, cudaStream_t stream) {
  if (n_del <= 0) return;
  DGNN_LAUNCH(k_deleted_contributor, wave_grid(n_del * w, 256, 8), 256, 0, stream, n_del, w,
              del_keys, argext, flag);
}

void agg_backward(int kind, int n, int w, const int64_t* out_ptr, const int32_t* out_dst,
                  const float* up, const float* degree, const int32_t* argext, float* grad,
                  cudaStream_t stream, const float* addend) {
  if (n <= 0 || w <= 0) return;
  const int vec = std::min(pick_vec(w, up, grad), pick_vec(w, addend, nullptr));
  if (kind == kAggSum && vec == 4 && !spmm_slicing_requested()) {
    if (const int U = spmm_u(w)) {
      launch_spmm_sum(U, n, w, out_ptr, out_dst, up, grad, addend, stream);
      return;
    }
  }
  const int wc = spmm_slice_width(n, w, vec);
  const int g = pick_group(wc, vec);
  const int grid = rows_grid(n, g);
  for (int c0 = 0; c0 < w; c0 += wc) {
    if (kind == kAggMean) {
      DGNN_DISPATCH_V(vec, DGNN_DISPATCH_G(g,
          DGNN_LAUNCH((k_agg_backward<V, G, true>), grid, kThreads, 0, stream, n, w, c0, wc,
                      out_ptr, out_dst, up, degree, grad, addend)));
    } else if (kind == kAggMax || kind == kAggMin) {
      DGNN_DISPATCH_V(vec, DGNN_DISPATCH_G(g,
          DGNN_LAUNCH((k_agg_backward<V, G, false, true>), grid, kThreads, 0, stream, n, w, c0, wc,
                      out_ptr, out_dst, up, degree, grad, addend, argext)));
    } else {
      DGNN_DISPATCH_V(vec, DGNN_DISPATCH_G(g,
          DGNN_LAUNCH((k_agg_backward<V, G, false>), grid, kThreads, 0, stream, n, w, c0, wc,
                      out_ptr, out_dst, up, degree, grad, addend)));
    }
  }
}

void mask_empty_rows(int n, int w, const int32_t* argext, const float* in, float* out,
                     cudaStream_t stream) {
  const int64_t total = static_cast<int64_t>(n) * w;
  if (total <= 0) return;
  DGNN_LAUNCH(k_mask_empty, wave_grid(total, 256, 8), 256, 0, stream, total, w, argext, in, out);
}

}  // namespace cuda
}  // namespace dgnn
