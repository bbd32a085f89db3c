// Dense kernels of the hot path for sm_100a.
//
// Round-1 implementation: FFMA (CUDA-core) tiles in fp32, one CTA owning all
// 4H gate columns of a row tile so the gate nonlinearities, the LSTM/GRU state
// update and the tape write are fused into the GEMM epilogue (no pre-activation
// round trip through HBM). Weight gradients use a fixed-order split over rows
// (partials + ordered reduction) so every run is bit-reproducible.
#include <algorithm>

#include "common.cuh"
#include "dense_kernels.h"

namespace dgnn {
namespace cuda {
namespace {

__device__ __forceinline__ float sigmoidf_(float x) { return 1.f / (1.f + expf(-x)); }

// ------------------------------------------------------------ cell forward
// Thread tile: RPT rows x (2 hidden units x 4 gate blocks). CG = H/2 column
// groups, RG = 256/CG row groups, BM = RG*RPT rows per CTA.
template <int H, int RPT, bool LSTM>
__global__ void __launch_bounds__(256)
k_cell_fwd(int n, int in, const float* __restrict__ X, const float* __restrict__ Hm,
           const float* __restrict__ hskip, const float* __restrict__ cprev,
           const float* __restrict__ W, const float* __restrict__ bias, float* __restrict__ gates,
           float* __restrict__ c_out, float* __restrict__ h_out) {
  constexpr int CG = H / 2;
  constexpr int RG = 256 / CG;
  constexpr int BM = RG * RPT;
  constexpr int NC = 4 * H;
  constexpr int KC = 16;
  __shared__ __align__(16) float As[KC][BM + 4];
  __shared__ __align__(16) float Bs[KC][NC];
  const int tid = threadIdx.x;
  const int cg = tid % CG;
  const int rg = tid / CG;
  const int K = in + H;
  for (int64_t r0 = static_cast<int64_t>(blockIdx.x) * BM; r0 < n;
       r0 += static_cast<int64_t>(gridDim.x) * BM) {
    float acc[RPT][8];
#pragma unroll
    for (int r = 0; r < RPT; ++r)
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[r][j] = 0.f;
    for (int k0 = 0; k0 < K; k0 += KC) {
      for (int i = tid; i < BM * KC; i += 256) {
        const int r = i / KC, kk = i % KC;
        const int k = k0 + kk;
        const int64_t row = r0 + r;
        float v = 0.f;
        if (row < n && k < K) v = k < in ? X[row * in + k] : Hm[row * H + (k - in)];
        As[kk][r] = v;
      }
      for (int i = tid; i < KC * NC; i += 256) {
        const int kk = i / NC, cc = i % NC;
        const int k = k0 + kk;
        Bs[kk][cc] = k < K ? W[static_cast<int64_t>(k) * NC + cc] : 0.f;
      }
      __syncthreads();
#pragma unroll
      for (int kk = 0; kk < KC; ++kk) {
        float a[RPT], b[8];
#pragma unroll
        for (int r = 0; r < RPT; ++r) a[r] = As[kk][rg * RPT + r];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float2 bb = *reinterpret_cast<const float2*>(&Bs[kk][q * H + cg * 2]);
          b[2 * q] = bb.x;
          b[2 * q + 1] = bb.y;
        }
#pragma unroll
        for (int r = 0; r < RPT; ++r)
#pragma unroll
          for (int j = 0; j < 8; ++j) acc[r][j] = fmaf(a[r], b[j], acc[r][j]);
      }
      __syncthreads();
    }
#pragma unroll
    for (int r = 0; r < RPT; ++r) {
      const int64_t row = r0 + rg * RPT + r;
      if (row >= n) continue;
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int j = cg * 2 + u;
        const float p0 = acc[r][0 + u] + bias[0 * H + j];
        const float p1 = acc[r][2 + u] + bias[1 * H + j];
        const float p2 = acc[r][4 + u];
        const float p3 = acc[r][6 + u];
        float* gr = gates + row * NC;
        if (LSTM) {
          const float ig = sigmoidf_(p0);
          const float fg = sigmoidf_(p1);
          const float gg = tanhf(p2 + bias[2 * H + j]);
          const float og = sigmoidf_(p3 + bias[3 * H + j]);
          const float c = fg * cprev[row * H + j] + ig * gg;
          gr[0 * H + j] = ig;
          gr[1 * H + j] = fg;
          gr[2 * H + j] = gg;
          gr[3 * H + j] = og;
          c_out[row * H + j] = c;
          h_out[row * H + j] = og * tanhf(c);
        } else {
          const float rr = sigmoidf_(p0);
          const float zz = sigmoidf_(p1);
          const float hn = p3;  // Hm * Uh_n, no bias (ref src/cells.cpp:123)
          const float nn = tanhf(p2 + rr * hn + bias[2 * H + j]);
          gr[0 * H + j] = rr;
          gr[1 * H + j] = zz;
          gr[2 * H + j] = nn;
          gr[3 * H + j] = hn;
          h_out[row * H + j] = (1.f - zz) * nn + zz * hskip[row * H + j];
        }
      }
    }
  }
}

// ------------------------------------------------------------ cell backward
template <bool LSTM>
__global__ void k_cell_bwd_pointwise(int64_t total, int H, const float* __restrict__ gates,
                                     const float* __restrict__ c, const float* __restrict__ cprev,
                                     const float* __restrict__ hskip, const float* __restrict__ dh,
                                     const float* __restrict__ dc, float* __restrict__ G,
                                     float* __restrict__ dc_prev, float* __restrict__ dh_skip) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t row = i / H;
    const int j = static_cast<int>(i - row * H);
    const float* gr = gates + row * 4 * H;
    float* go = G + row * 4 * H;
    const float d = dh[i];
    if (LSTM) {
      const float ig = gr[j], fg = gr[H + j], gg = gr[2 * H + j], og = gr[3 * H + j];
      const float tc = tanhf(c[i]);
      const float d_o = d * tc;
      float dct = (1.f - tc * tc) * (d * og);
      if (dc) dct += dc[i];
      const float d_i = dct * gg, d_g = dct * ig, d_f = dct * cprev[i];
      dc_prev[i] = dct * fg;
      go[j] = ig * (1.f - ig) * d_i;
      go[H + j] = fg * (1.f - fg) * d_f;
      go[2 * H + j] = (1.f - gg * gg) * d_g;
      go[3 * H + j] = og * (1.f - og) * d_o;
    } else {
      const float rr = gr[j], zz = gr[H + j], nn = gr[2 * H + j], hn = gr[3 * H + j];
      const float d_z = d * (hskip[i] - nn);
      const float d_n = d * (1.f - zz);
      dh_skip[i] = d * zz;
      const float dpre_n = (1.f - nn * nn) * d_n;
      const float d_hn = dpre_n * rr;
      const float d_r = dpre_n * hn;
      go[j] = rr * (1.f - rr) * d_r;
      go[H + j] = zz * (1.f - zz) * d_z;
      go[2 * H + j] = dpre_n;
      go[3 * H + j] = d_hn;
    }
  }
}

// ------------------------------------------------------------ generic GEMMs
constexpr int TB = 64, TK = 16;

__global__ void __launch_bounds__(256)
k_gemm_nn(int m, int k1, int k2, int n1, int n2, const float* __restrict__ A1,
          const float* __restrict__ A2, const float* __restrict__ B, int ldb,
          const float* __restrict__ bias,
          int relu, int accumulate, float* __restrict__ C1, float* __restrict__ C2) {
  __shared__ __align__(16) float As[TK][TB + 4];
  __shared__ __align__(16) float Bs[TK][TB];
  const int tid = threadIdx.x, tx = tid % 16, ty = tid / 16;
  const int K = k1 + k2, N = n1 + n2;
  const int64_t r0 = static_cast<int64_t>(blockIdx.y) * TB;
  const int c0 = blockIdx.x * TB;
  float acc[4][4] = {};
  for (int k0 = 0; k0 < K; k0 += TK) {
    for (int i = tid; i < TB * TK; i += 256) {
      const int r = i / TK, kk = i % TK, k = k0 + kk;
      const int64_t row = r0 + r;
      float v = 0.f;
      if (row < m && k < K) v = k < k1 ? A1[row * k1 + k] : A2[row * k2 + (k - k1)];
      As[kk][r] = v;
    }
    for (int i = tid; i < TB * TK; i += 256) {
      const int kk = i / TB, cc = i % TB, k = k0 + kk, c = c0 + cc;
      Bs[kk][cc] = (k < K && c < N) ? B[static_cast<int64_t>(k) * ldb + c] : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < TK; ++kk) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t row = r0 + ty * 4 + i;
    if (row >= m) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int c = c0 + tx * 4 + j;
      if (c >= N) continue;
      float v = acc[i][j];
      if (bias) v += bias[c];
      if (relu) v = v > 0.f ? v : 0.f;
      float* dst = c < n1 ? C1 + row * n1 + c : C2 + row * n2 + (c - n1);
      *dst = accumulate ? *dst + v : v;
    }
  }
}

// Partial D_s = A[rows of slice s]^T * B[rows of slice s] for one 64x64 tile.
__global__ void __launch_bounds__(256)
k_gemm_tn_partial(int m, int k1, int k2, int nc, int slices, const float* __restrict__ A1,
                  const float* __restrict__ A2, const float* __restrict__ B, int nb,
                  float* __restrict__ ws, float* __restrict__ wsb) {
  __shared__ __align__(16) float As[TK][TB];
  __shared__ __align__(16) float Bs[TK][TB];
  const int tid = threadIdx.x, tx = tid % 16, ty = tid / 16;
  const int K = k1 + k2;
  const int kt0 = blockIdx.y * TB, ct0 = blockIdx.x * TB;
  const int s = blockIdx.z;
  const int64_t rows_per = (m + slices - 1) / slices;
  const int64_t rb = s * rows_per, re = min(static_cast<int64_t>(m), rb + rows_per);
  float acc[4][4] = {};
  float bsum = 0.f;  // column sum (k tile 0, one column per thread < TB)
  for (int64_t q0 = rb; q0 < re; q0 += TK) {
    for (int i = tid; i < TB * TK; i += 256) {
      const int rr = i / TB, kk = i % TB;
      const int64_t row = q0 + rr;
      const int k = kt0 + kk;
      float v = 0.f;
      if (row < re && k < K) v = k < k1 ? A1[row * k1 + k] : A2[row * k2 + (k - k1)];
      As[rr][kk] = v;
      const int c = ct0 + kk;
      Bs[rr][kk] = (row < re && c < nc) ? B[row * nc + c] : 0.f;
    }
    __syncthreads();
    if (blockIdx.y == 0 && tid < TB) {
#pragma unroll
      for (int rr = 0; rr < TK; ++rr) bsum += Bs[rr][tid];
    }
#pragma unroll
    for (int rr = 0; rr < TK; ++rr) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[rr][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[rr][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
  float* out = ws + static_cast<int64_t>(s) * K * nc;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int k = kt0 + ty * 4 + i;
    if (k >= K) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int c = ct0 + tx * 4 + j;
      if (c < nc) out[static_cast<int64_t>(k) * nc + c] = acc[i][j];
    }
  }
  if (blockIdx.y == 0 && tid < TB && ct0 + tid < nb) wsb[static_cast<int64_t>(s) * nb + ct0 + tid] = bsum;
}

__global__ void k_reduce_slices(int64_t len, int slices, const float* __restrict__ ws,
                                float* __restrict__ D) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < len;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    float acc = 0.f;
    for (int s = 0; s < slices; ++s) acc += ws[s * len + i];
    D[i] += acc;
  }
}

__global__ void k_transpose(int rows, int cols, const float* __restrict__ in, float* __restrict__ out) {
  const int64_t total = static_cast<int64_t>(rows) * cols;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = i / cols;
    const int c = static_cast<int>(i - r * cols);
    out[static_cast<int64_t>(c) * rows + r] = in[i];
  }
}

__global__ void k_relu_bwd(int64_t n, const float* __restrict__ out, const float* __restrict__ dout,
                           float* __restrict__ dpre) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    dpre[i] = out[i] > 0.f ? dout[i] : 0.f;
}

__global__ void k_axpy(int64_t n, float alpha, const float* __restrict__ x, float* __restrict__ y) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    y[i] += alpha * x[i];
}

// ------------------------------------------------------------ loss
constexpr int kLossBlocks = 296;

__global__ void __launch_bounds__(256)
k_mae(int n, int d, int r0, int r1, const float* __restrict__ pred, const float* __restrict__ target,
      float* __restrict__ dpred, float gscale, double* __restrict__ ws) {
  __shared__ double red[256];
  const int64_t total = static_cast<int64_t>(n) * d;
  const int64_t lo = static_cast<int64_t>(r0) * d, hi = static_cast<int64_t>(r1) * d;
  double acc = 0.0;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    float g = 0.f;
    if (i >= lo && i < hi) {
      const float diff = pred[i] - target[i];
      acc += fabs(static_cast<double>(diff));
      g = diff > 0.f ? gscale : (diff < 0.f ? -gscale : 0.f);
    }
    dpred[i] = g;
  }
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int s = 128; s > 0; s >>= 1) {
    if (threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) ws[blockIdx.x] = red[0];
}

// 128-bit variant (d % 4 == 0, aligned): four float4 pairs in flight per
// thread per iteration — the scalar loop left too few bytes in flight to
// stream 2 x 2 GB at C4 (4 ms per call, now bandwidth-bound).
__global__ void __launch_bounds__(512)
k_mae4(int64_t total4, int d4, int64_t lo4, int64_t hi4, const float4* __restrict__ pred,
       const float4* __restrict__ target, float4* __restrict__ dpred, float gscale,
       double* __restrict__ ws) {
  __shared__ double red[512];
  double acc = 0.0;
  constexpr int U = 4;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i0 = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i0 < total4;
       i0 += stride * U) {
    float4 pv[U], tv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = i0 + u * stride;
      if (i < total4) {
        pv[u] = __ldg(pred + i);
        tv[u] = __ldg(target + i);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = i0 + u * stride;
      if (i >= total4) continue;
      float4 g = make_float4(0.f, 0.f, 0.f, 0.f);
      if (i >= lo4 && i < hi4) {
        const float dx = pv[u].x - tv[u].x, dy = pv[u].y - tv[u].y;
        const float dz = pv[u].z - tv[u].z, dw = pv[u].w - tv[u].w;
        acc += fabs(static_cast<double>(dx)) + fabs(static_cast<double>(dy)) +
               fabs(static_cast<double>(dz)) + fabs(static_cast<double>(dw));
        auto sg = [&](float v) { return v > 0.f ? gscale : (v < 0.f ? -gscale : 0.f); };
        g = make_float4(sg(dx), sg(dy), sg(dz), sg(dw));
      }
      dpred[i] = g;
    }
  }
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int s = 256; s > 0; s >>= 1) {
    if (threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) ws[blockIdx.x] = red[0];
  (void)d4;
}

__global__ void k_mae_finish(int nblocks, const double* __restrict__ ws, double scale,
                             double* __restrict__ loss_out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double s = 0.0;
    for (int b = 0; b < nblocks; ++b) s += ws[b];
    *loss_out += s * scale;
  }
}

__global__ void k_nonfinite(int64_t n, const float* __restrict__ x, int32_t* flag) {
  int bad = 0;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    bad |= !isfinite(x[i]);
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flag, 1);
}

__global__ void k_adam(int64_t n, float* __restrict__ p, float* __restrict__ m, float* __restrict__ v,
                       const float* __restrict__ g, float gscale, float lr, float b1, float b2,
                       float eps, float bc1, float bc2, int sgd, const int32_t* __restrict__ skip) {
  if (skip && *skip) return;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const float gi = g[i] * gscale;
    if (sgd) {
      p[i] -= lr * gi;
      continue;
    }
    const float mi = b1 * m[i] + (1.f - b1) * gi;
    const float vi = b2 * v[i] + (1.f - b2) * gi * gi;
    m[i] = mi;
    v[i] = vi;
    p[i] -= lr * (mi / bc1) / (sqrtf(vi / bc2) + eps);
  }
}

// ------------------------------------------------------------ packing
__global__ void k_pack_cell(int lstm, int in, int H, const float* __restrict__ flat,
                            float* __restrict__ W, float* __restrict__ bias) {
  const int K = in + H, NC = 4 * H;
  const int gates = lstm ? 4 : 3;
  const int64_t per_gate = static_cast<int64_t>(in) * H + static_cast<int64_t>(H) * H + H;
  const int64_t total = static_cast<int64_t>(K) * NC + NC;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    if (i < static_cast<int64_t>(K) * NC) {
      const int k = static_cast<int>(i / NC), col = static_cast<int>(i % NC);
      const int q = col / H, j = col % H;
      float v = 0.f;
      // gate providing this block's X rows / Hm rows (-1: zero block)
      const int gx = lstm ? q : (q == 3 ? -1 : q);
      const int gh = lstm ? q : (q == 2 ? -1 : (q == 3 ? 2 : q));
      if (k < in) {
        if (gx >= 0) v = flat[gx * per_gate + static_cast<int64_t>(k) * H + j];
      } else if (gh >= 0) {
        v = flat[gh * per_gate + static_cast<int64_t>(in) * H + static_cast<int64_t>(k - in) * H + j];
      }
      W[i] = v;
    } else {
      const int col = static_cast<int>(i - static_cast<int64_t>(K) * NC);
      const int q = col / H, j = col % H;
      const int gb = q < gates ? q : -1;
      bias[col] = gb >= 0 ? flat[gb * per_gate + static_cast<int64_t>(in) * H +
                                 static_cast<int64_t>(H) * H + j]
                          : 0.f;
    }
  }
}

__global__ void k_unpack_cell_grad(int lstm, int in, int H, const float* __restrict__ dW,
                                   const float* __restrict__ db, float* __restrict__ flat) {
  const int gates = lstm ? 4 : 3;
  const int NC = 4 * H;
  const int64_t per_gate = static_cast<int64_t>(in) * H + static_cast<int64_t>(H) * H + H;
  const int64_t total = per_gate * gates;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int g = static_cast<int>(i / per_gate);
    int64_t o = i - g * per_gate;
    float v;
    if (o < static_cast<int64_t>(in) * H) {  // wx_g
      const int k = static_cast<int>(o / H), j = static_cast<int>(o % H);
      v = dW[static_cast<int64_t>(k) * NC + g * H + j];
    } else if ((o -= static_cast<int64_t>(in) * H) < static_cast<int64_t>(H) * H) {  // uh_g
      const int k = static_cast<int>(o / H), j = static_cast<int>(o % H);
      const int q = lstm ? g : (g == 2 ? 3 : g);
      v = dW[static_cast<int64_t>(in + k) * NC + q * H + j];
    } else {  // b_g
      const int j = static_cast<int>(o - static_cast<int64_t>(H) * H);
      v = db[g * H + j];
    }
    flat[i] += v;
  }
}

template <int H, int RPT, bool LSTM>
void launch_cell_fwd(int n, int in, const float* X, const float* Hm, const float* hs,
                     const float* cp, const float* W, const float* b, float* gates, float* c,
                     float* h, cudaStream_t st) {
  constexpr int BM = (256 / (H / 2)) * RPT;
  const int grid = wave_grid((static_cast<int64_t>(n) + BM - 1) / BM * 256, 256, 2);
  DGNN_LAUNCH((k_cell_fwd<H, RPT, LSTM>), grid, 256, 0, st, n, in, X, Hm, hs, cp, W, b, gates, c, h);
}

}  // namespace

void cell_forward(bool lstm, int n, int in, int H, const float* X, const float* Hm,
                  const float* h_skip, const float* c_prev, const float* W, const float* bias,
                  float* gates, float* c, float* h, cudaStream_t stream) {
  if (n <= 0) return;
#define DGNN_CELL_CASE(HH, RPT)                                                                 \
  case HH:                                                                                      \
    if (lstm)                                                                                   \
      launch_cell_fwd<HH, RPT, true>(n, in, X, Hm, h_skip, c_prev, W, bias, gates, c, h, stream); \
    else                                                                                        \
      launch_cell_fwd<HH, RPT, false>(n, in, X, Hm, h_skip, c_prev, W, bias, gates, c, h, stream); \
    break;
  switch (H) {
    DGNN_CELL_CASE(8, 2)
    DGNN_CELL_CASE(16, 4)
    DGNN_CELL_CASE(32, 8)
    DGNN_CELL_CASE(64, 8)
    DGNN_CELL_CASE(128, 8)
    default:
      throw std::invalid_argument("cell_forward: hidden_dim must be one of 8,16,32,64,128 (got " +
                                  std::to_string(H) + ")");
  }
#undef DGNN_CELL_CASE
}

void cell_backward_pointwise(bool lstm, int n, int H, const float* gates, const float* c,
                             const float* c_prev, const float* h_skip, const float* dh,
                             const float* dc, float* G, float* dc_prev, float* dh_skip,
                             cudaStream_t stream) {
  const int64_t total = static_cast<int64_t>(n) * H;
  if (total <= 0) return;
  const int grid = wave_grid(total, 256, 8);
  if (lstm) {
    DGNN_LAUNCH(k_cell_bwd_pointwise<true>, grid, 256, 0, stream, total, H, gates, c, c_prev,
                h_skip, dh, dc, G, dc_prev, dh_skip);
  } else {
    DGNN_LAUNCH(k_cell_bwd_pointwise<false>, grid, 256, 0, stream, total, H, gates, c, c_prev,
                h_skip, dh, dc, G, dc_prev, dh_skip);
  }
}

void gemm_nn(int m, int k1, int k2, int n1, int n2, const float* A1, const float* A2,
             const float* B, int ldb, const float* bias, bool relu, bool accumulate, float* C1,
             float* C2, cudaStream_t stream) {
  if (m <= 0 || n1 + n2 <= 0) return;
  dim3 grid(ceil_div(n1 + n2, TB), ceil_div(m, TB));
  DGNN_LAUNCH(k_gemm_nn, grid, 256, 0, stream, m, k1, k2, n1, n2, A1, A2, B, ldb, bias,
              relu ? 1 : 0, accumulate ? 1 : 0, C1, C2);
}

void relu_backward(int64_t n, const float* out, const float* dout, float* dpre,
                   cudaStream_t stream) {
  if (n <= 0) return;
  DGNN_LAUNCH(k_relu_bwd, wave_grid(n, 256, 8), 256, 0, stream, n, out, dout, dpre);
}

namespace {
int tn_slices(int m, int k, int nc) {
  const int tiles = ceil_div(k, TB) * ceil_div(nc, TB);
  int s = ceil_div(2 * kNumSMs, tiles);
  const int max_s = ceil_div(m, 256);
  if (s > max_s) s = max_s;
  return s < 1 ? 1 : s;
}
}  // namespace

int64_t gemm_tn_workspace(int m, int k, int nc) {
  const int s = tn_slices(m, k, nc);
  return static_cast<int64_t>(s) * k * nc + static_cast<int64_t>(s) * nc;
}

void gemm_tn_acc(int m, int k1, int k2, int nc, const float* A1, const float* A2, const float* B,
                 float* D, int nb, float* bias_grad, float* ws, cudaStream_t stream) {
  const int K = k1 + k2;
  if (m <= 0 || K <= 0 || nc <= 0) return;
  const int s = tn_slices(m, K, nc);
  float* wsb = ws + static_cast<int64_t>(s) * K * nc;
  const int nbv = bias_grad ? nb : 0;
  dim3 grid(ceil_div(nc, TB), ceil_div(K, TB), s);
  DGNN_LAUNCH(k_gemm_tn_partial, grid, 256, 0, stream, m, k1, k2, nc, s, A1, A2, B, nbv, ws, wsb);
  const int64_t len = static_cast<int64_t>(K) * nc;
  DGNN_LAUNCH(k_reduce_slices, wave_grid(len, 256, 4), 256, 0, stream, len, s, ws, D);
  if (nbv > 0)
    DGNN_LAUNCH(k_reduce_slices, wave_grid(nbv, 256, 4), 256, 0, stream, static_cast<int64_t>(nbv),
                s, wsb, bias_grad);
}

void transpose(int rows, int cols, const float* in, float* out, cudaStream_t stream) {
  const int64_t total = static_cast<int64_t>(rows) * cols;
  if (total <= 0) return;
  DGNN_LAUNCH(k_transpose, wave_grid(total, 256, 4), 256, 0, stream, rows, cols, in, out);
}

void axpy(int64_t n, float alpha, const float* x, float* y, cudaStream_t stream) {
  if (n <= 0) return;
  DGNN_LAUNCH(k_axpy, wave_grid(n, 256, 8), 256, 0, stream, n, alpha, x, y);
}

void mae_loss(int n, int d, int r0, int r1, const float* pred, const float* target, float* dpred,
              double inv_h, double* loss_out, double* ws, cudaStream_t stream) {
  const double n_el = static_cast<double>(r1 - r0) * d;
  const float gscale = static_cast<float>(1.0 / n_el * inv_h);
  auto al16 = [](const void* q) { return (reinterpret_cast<uintptr_t>(q) & 15) == 0; };
  if (d % 4 == 0 && al16(pred) && al16(target) && al16(dpred)) {
    const int64_t d4 = d / 4;
    DGNN_LAUNCH(k_mae4, kLossBlocks, 512, 0, stream, static_cast<int64_t>(n) * d4, static_cast<int>(d4),
                r0 * d4, r1 * d4, reinterpret_cast<const float4*>(pred),
                reinterpret_cast<const float4*>(target), reinterpret_cast<float4*>(dpred), gscale, ws);
  } else {
    DGNN_LAUNCH(k_mae, kLossBlocks, 256, 0, stream, n, d, r0, r1, pred, target, dpred, gscale, ws);
  }
  DGNN_LAUNCH(k_mae_finish, 1, 32, 0, stream, kLossBlocks, ws, inv_h / n_el, loss_out);
}

void nonfinite_check(int64_t n, const float* x, int32_t* flag, cudaStream_t stream) {
  if (n <= 0) return;
  DGNN_LAUNCH(k_nonfinite, wave_grid(n, 256, 4), 256, 0, stream, n, x, flag);
}

void adam_step(int64_t n, float* p, float* m, float* v, const float* g, float gscale, float lr,
               float beta1, float beta2, float eps, float bc1, float bc2, bool sgd,
               const int32_t* skip_flag, cudaStream_t stream) {
  if (n <= 0) return;
  DGNN_LAUNCH(k_adam, wave_grid(n, 256, 4), 256, 0, stream, n, p, m, v, g, gscale, lr, beta1,
              beta2, eps, bc1, bc2, sgd ? 1 : 0, skip_flag);
}

void pack_cell(bool lstm, int in, int H, const float* flat, float* W, float* bias,
               cudaStream_t stream) {
  const int64_t total = static_cast<int64_t>(in + H) * 4 * H + 4 * H;
  DGNN_LAUNCH(k_pack_cell, wave_grid(total, 256, 4), 256, 0, stream, lstm ? 1 : 0, in, H, flat, W,
              bias);
}

namespace {
// all cells of a model in one launch (blockIdx.y = cell)
__global__ void k_zero_cells(const CellGradDesc* __restrict__ cells, int n) {
  const CellGradDesc c = cells[blockIdx.y];
  const int64_t nw = static_cast<int64_t>(c.in + c.H) * 4 * c.H, nb = 4 * c.H;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < nw + nb;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    if (i < nw) c.dW[i] = 0.f;
    else c.db[i - nw] = 0.f;
  }
  (void)n;
}

__global__ void k_unpack_cells(const CellGradDesc* __restrict__ cells, float* __restrict__ flat) {
  const CellGradDesc c = cells[blockIdx.y];
  const int lstm = c.lstm, in = c.in, H = c.H;
  const int gates = lstm ? 4 : 3;
  const int NC = 4 * H;
  const int64_t per_gate = static_cast<int64_t>(in) * H + static_cast<int64_t>(H) * H + H;
  const int64_t total = per_gate * gates;
  float* out = flat + c.offset;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int g = static_cast<int>(i / per_gate);
    int64_t o = i - g * per_gate;
    float v;
    if (o < static_cast<int64_t>(in) * H) {
      const int k = static_cast<int>(o / H), j = static_cast<int>(o % H);
      v = c.dW[static_cast<int64_t>(k) * NC + g * H + j];
    } else if ((o -= static_cast<int64_t>(in) * H) < static_cast<int64_t>(H) * H) {
      const int k = static_cast<int>(o / H), j = static_cast<int>(o % H);
      const int q = lstm ? g : (g == 2 ? 3 : g);
      v = c.dW[static_cast<int64_t>(in + k) * NC + q * H + j];
    } else {
      const int j = static_cast<int>(o - static_cast<int64_t>(H) * H);
      v = c.db[g * H + j];
    }
    out[i] += v;
  }
}
}  // namespace

void zero_cell_grads(const CellGradDesc* cells_dev, int n, int64_t max_elems, cudaStream_t stream) {
  if (n <= 0) return;
  const dim3 grid(static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>((max_elems + 255) / 256, 256))),
                  static_cast<unsigned>(n));
  DGNN_LAUNCH(k_zero_cells, grid, 256, 0, stream, cells_dev, n);
}

void unpack_cell_grads(const CellGradDesc* cells_dev, int n, int64_t max_elems, float* flat_grad,
                       cudaStream_t stream) {
  if (n <= 0) return;
  const dim3 grid(static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>((max_elems + 255) / 256, 256))),
                  static_cast<unsigned>(n));
  DGNN_LAUNCH(k_unpack_cells, grid, 256, 0, stream, cells_dev, flat_grad);
}

void unpack_cell_grad(bool lstm, int in, int H, const float* dW, const float* db,
                      float* flat_grad, cudaStream_t stream) {
  const int64_t total = (static_cast<int64_t>(in) * H + static_cast<int64_t>(H) * H + H) * (lstm ? 4 : 3);
  DGNN_LAUNCH(k_unpack_cell_grad, wave_grid(total, 256, 4), 256, 0, stream, lstm ? 1 : 0, in, H,
              dW, db, flat_grad);
}

}  // namespace cuda
}  // namespace dgnn
