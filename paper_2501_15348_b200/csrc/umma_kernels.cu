// tcgen05 (5th-gen tensor core) kernels for the dense part of the GraphRNN
// cell, fp32-accurate through a 3xTF32 split:
//   a*b ~= a_hi*b_hi + a_hi*b_lo + a_lo*b_hi  (kind::tf32, fp32 accumulate in TMEM)
//
//   k_row_gemm  D[128-row tile x N] = [A1|A2](rows x K) * B^T, B = packed
//               weight image (N x K, K-major), with a fused epilogue:
//               LSTM / GRU gates + state update + tape write (cell forward),
//               or a column-split store (cell backward dX | dHm).
//   k_wgrad     per-CTA partial of G^T * [X | Hm | 1] over a contiguous row
//               range (weight + bias gradients), reduced in fixed CTA order.
//
// k_row_gemm is a persistent, warp-specialised kernel (one CTA per SM):
//   warps 0-3  producers: A tile global -> registers -> 3xTF32 split -> smem
//              (canonical K-major UMMA layout); the leader also issues the
//              bulk (TMA-engine) copy of the pre-split B chunk;
//   warp 4     TMEM allocator + the single thread issuing tcgen05.mma;
//   warps 5-12 epilogue: tcgen05.ld from TMEM, fused math, stores coalesced
//              through a per-warp smem transpose (8 rows x 64 B per store).
// Smem stages (4 x K=16) are handed over with full/empty mbarriers
// (expect_tx for the bulk copy, tcgen05.commit for release); the fp32
// accumulator is double-buffered in TMEM (2 x 256 columns) so the epilogue of
// tile i overlaps the MMAs of tile i+1.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <string>
#include <type_traits>

#include "common.cuh"
#include "umma.cuh"
#include "umma_kernels.h"

namespace dgnn {
namespace cuda {
namespace {

using namespace umma;

constexpr int kTileM = 128;  // rows per MMA tile (cta_group::1, M = 128)
constexpr int kKC = 16;      // K elements per staged chunk (2 MMA K-steps of 8)

// Epilogue transcendentals on the SFU (__expf: 2 ulp) with well-conditioned
// forms: absolute error ~1e-7 on O(1) gate values, far inside the 1e-5
// norm-relative tape tolerance, at a fraction of the libm instruction count.
__device__ __forceinline__ float sigm(float x) { return __fdividef(1.f, 1.f + __expf(-x)); }
__device__ __forceinline__ float ftanh(float x) {
  const float e = __expf(-2.f * fabsf(x));
  return copysignf(__fdividef(1.f - e, 1.f + e), x);
}
__device__ __forceinline__ void st_shared_v4(uint32_t addr, float a, float b, float c, float d) {
  asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "f"(a), "f"(b), "f"(c), "f"(d)
               : "memory");
}

// ------------------------------------------------------------- B images
// out: per K chunk c: [hi tile (Npad x KC)][lo tile], canonical layout.
// B(n, k) = trans ? M[k * ld + (n0 + n)] : M[(n0 + n) * ld + k]; zero padded.
// perm_h > 0: GRU column blocks stored as [n | r | z | hn] (source blocks
// r, z, n, hn = 0..3 of width perm_h), see RowGemmArgs::gru_split.
__global__ void k_pack_b(const float* __restrict__ M, int ld, int trans, int n0, int N, int K,
                         int Npad, int nchunks, float* __restrict__ out, int perm_h) {
  const int64_t per_tile = tile_bytes(Npad, kKC) / 4;
  const int64_t total = static_cast<int64_t>(nchunks) * Npad * kKC;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int c = static_cast<int>(i / (static_cast<int64_t>(Npad) * kKC));
    const int rem = static_cast<int>(i - static_cast<int64_t>(c) * Npad * kKC);
    const int n = rem / kKC, kk = rem % kKC;
    const int k = c * kKC + kk;
    int ns = n;
    if (perm_h > 0 && n < N) {
      const int blk = n / perm_h;
      ns = (blk == 0 ? 2 : (blk == 3 ? 3 : blk - 1)) * perm_h + n % perm_h;
    }
    float v = 0.f;
    if (n < N && k < K) v = trans ? M[static_cast<int64_t>(k) * ld + n0 + ns] : M[static_cast<int64_t>(n0 + ns) * ld + k];
    float hi, lo;
    split_tf32(v, hi, lo);
    float* base = out + static_cast<int64_t>(c) * 2 * per_tile;
    const uint32_t off = tile_offset(Npad, n, kk) / 4;
    base[off] = hi;
    base[per_tile + off] = lo;
  }
}

// ------------------------------------------------------------- row GEMM
// kEpiLstmBwd / kEpiGruBwd recompute the forward gates from the same operands
// (bit-identical to the forward epilogue: same MMA order, same math) and
// apply the pointwise cell backward (ref src/cells.cpp:134-166) in place of a
// gates tape: the forward then stores only its state, the backward reads
// X | Hm instead of the 4H-wide gates (+ c).
enum { kEpiLstm = 0, kEpiGru = 1, kEpiStore2 = 2, kEpiLstmBwd = 3, kEpiGruBwd = 4 };

template <int EPI>
constexpr bool kEpiCell = EPI == kEpiLstm || EPI == kEpiGru || EPI == kEpiLstmBwd || EPI == kEpiGruBwd;
template <int EPI>
constexpr bool kEpiLstmLike = EPI == kEpiLstm || EPI == kEpiLstmBwd;

struct RowGemmArgs {
  int M, k1, k2, K, nchunks;
  const float* A1;
  const float* A2;
  const float* Bimg;
  // cell epilogue
  int H;
  const float* bias;
  const float* c_prev;
  const float* h_skip;
  float* gates;  // may be null (recompute mode: no gates tape)
  float* c_out;
  float* h_out;
  // backward cell epilogue: upstream dh (dc), outputs G (n x 4H) and
  // dstate = dc_prev (LSTM) / dh_skip (GRU)
  const float* dh;
  const float* dc;
  float* G;
  float* dstate;
  // store2 epilogue (optional bias over C1's columns, C1 += result)
  int n1, n2;
  float* C1;
  float* C2;
  int store_accumulate;
  int relu;  // store2: C1 = max(C1, 0) after bias / accumulate (the GCN layer's ReLU)
  // GRU block-sparse contraction (0 = off, else H): the B image holds the
  // gate columns as [n | r | z | hn]; X-only K chunks skip the hn block
  // (X has no h-part of the candidate gate) and Hm-only chunks skip the
  // x-part n block, i.e. N = 3H instead of 4H after a full-N first chunk
  // that initialises every accumulator column.
  int gru_split;
  // GRU block sparsity of the store2 contraction G . W^T (0 = off, else H):
  // K chunks of the n block feed only the x columns [0, s2_nx), chunks of
  // the hn block only the h columns [s2_h0, s2_h0 + H); r / z chunks all.
  int s2_gru, s2_nx, s2_h0;
  // cell epilogues: the hi*hi products accumulate in TMEM columns [0, 256)
  // and the two correction products in [256, 512), summed (RN) in the
  // epilogue. The tensor core adds into its fp32 accumulator with truncation,
  // and that bias grows with every accumulate into a large-magnitude sum:
  // keeping the 2/3 of the MMAs that carry the small correction terms out of
  // the big accumulator cuts the pre-activation error ~3x (measured against
  // the fp64 reference on C4-shaped cells). Costs the TMEM double buffer.
  // (Measured alternative with the same accuracy and no extra TMEM: two
  // passes over K per tile, corrections first, then hi*hi — the same ~40%
  // forward-kernel cost from re-reading / re-splitting A, and slower in the
  // C4 epoch, so not kept.)
  int split_acc;
  // A rows are not 16 B multiples (k1 % 4 or k2 % 4 != 0): element copies
  int scalar_a;
  // profiling switches (env DGNN_UMMA_DEBUG): 1 skip epilogue math/stores,
  // 2 skip the B copy, 4 skip the A split/stores
  int debug;
};

// DGNN_SPLIT_ACC bit 1: cell forward, bit 2: backward gate recompute. The
// forward's split sets the accuracy of h / predictions (and through them the
// gradients); splitting the recompute as well measured no further gain on
// the C4-shaped gradients and costs ~0.7 s per C4 epoch, so it is off.
int umma_split_acc() {
  static const int v = [] {
    const char* e = std::getenv("DGNN_SPLIT_ACC");
    return e ? std::atoi(e) : 1;
  }();
  return v;
}

int umma_debug_flags() {
  static const int f = [] {
    const char* e = std::getenv("DGNN_UMMA_DEBUG");
    return e ? std::atoi(e) : 0;
  }();
  return f;
}

#ifndef DGNN_RG_PRODUCER_WARPS
#define DGNN_RG_PRODUCER_WARPS 4
#endif
// warps: producers, 1 MMA, 8 epilogue
constexpr int kProducerWarps = DGNN_RG_PRODUCER_WARPS;
constexpr int kRgThreads = 32 * (kProducerWarps + 1 + 8);
// MMA operand stages (A hi/lo + B hi/lo): the producer -> tcgen05 -> commit
// round trip is latency-bound (ncu: producers wait on `empty`, the MMA thread
// on `full`, the tensor pipe < 20% busy), so small-N contractions get more
// stages in the smem their smaller B tiles leave free
template <int NPAD>
constexpr int kRgStagesFor = NPAD <= 64 ? 6 : (NPAD <= 128 ? 5 : (NPAD <= 192 ? 4 : 3));
// cp.async prefetch depth of raw fp32 A chunks: as deep as shared memory
// allows (the producers are latency-bound on 128 separate 64 B row segments
// per chunk; small-N contractions have little MMA work to hide it behind)
template <int NPAD>
constexpr int kRawSlotsFor = NPAD <= 64 ? 7 : (NPAD <= 192 ? 5 : 6);
constexpr int kProducerThreads = 32 * kProducerWarps;
constexpr int kProducerRows = kProducerThreads / 4;  // rows per producer pass (4 K quads per row)
constexpr int kMmaWarp = kProducerWarps;
// 8 epilogue warps: lane quadrant = warp % 4 covers 0..3 twice
constexpr int kEpiWarp0 = kProducerWarps + 1;
constexpr int kEpiWarps = 8;
constexpr int kRawPerThread = (kTileM * kKC / 4) / kProducerThreads;  // float4 per thread per chunk

template <int NPAD>
struct RowGemmSmem {
  static constexpr uint32_t kA = tile_bytes(kTileM, kKC);  // one A tile (hi or lo)
  static constexpr uint32_t kB = tile_bytes(NPAD, kKC);
  static constexpr uint32_t kStage = 2 * kA + 2 * kB;
  static constexpr uint32_t kRaw = kTileM * kKC * 4;      // one raw fp32 A chunk
  static constexpr int kStages = kRgStagesFor<NPAD>;
  static constexpr uint32_t kRawOff = kStage * kStages;
  static constexpr int kRawSlots = kRawSlotsFor<NPAD>;
  static constexpr uint32_t kBars = kRawOff + kRaw * kRawSlots;  // barrier block offset
  static constexpr uint32_t kBias = kBars + 256;                 // 4H fp32 bias copy
  static constexpr uint32_t kOut = kBias + 1024;                 // per-epilogue-warp store staging
  static constexpr uint32_t kBytes = kOut + kEpiWarps * 32 * 16 * 4;
};

__device__ __forceinline__ void cp_async16_zfill(uint32_t saddr, const void* g, bool valid) {
  const int n = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(saddr), "l"(g), "r"(n) : "memory");
}
// 4-byte element copy (operands whose rows are not 16 B multiples)
__device__ __forceinline__ void cp_async4_zfill(uint32_t saddr, const void* g, bool valid) {
  const int n = valid ? 4 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(saddr), "l"(g), "r"(n) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

template <int EPI, int NPAD>
__global__ void __launch_bounds__(kRgThreads, 1) k_row_gemm(RowGemmArgs p) {
  using S = RowGemmSmem<NPAD>;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S::kBars);
  uint64_t* empty = full + S::kStages;
  uint64_t* tfull = empty + S::kStages;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (warp == kMmaWarp) tmem_alloc(tmem_slot, 512);
  if (tid == 0) {
    for (int s = 0; s < S::kStages; ++s) {
      mbar_init(&full[s], kProducerThreads);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], kEpiWarps);
    }
    fence_barrier_init();
  }
  float* sbias = reinterpret_cast<float*>(smem + S::kBias);
  if (kEpiCell<EPI> && tid < 4 * p.H) sbias[tid] = p.bias[tid];
  if (EPI == kEpiStore2 && p.bias != nullptr && tid < p.n1) sbias[tid] = p.bias[tid];
  fence_before_sync();
  __syncthreads();
  fence_after_sync();
  const uint32_t tmem = *tmem_slot;
  const uint32_t sbase = smem_u32(smem);
  const int ntiles = (p.M + kTileM - 1) / kTileM;

  if (warp < kProducerWarps) {
    // ---------------- producers
    // Flat sequence of (tile, chunk) items; raw fp32 A chunks are prefetched
    // kRawSlots - 1 items ahead with cp.async (each thread later re-reads only
    // what it copied, so no cross-thread sync is needed before the split).
    const int my_tiles = blockIdx.x < ntiles ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    const int total = my_tiles * p.nchunks;
    const uint32_t raw0 = sbase + S::kRawOff;
    // This thread's units of every chunk: rows prow + 32 * it, K quad kq
    // (f = tid + 128 * it). Issue / consume positions are advanced
    // incrementally — no per-item integer division (the producers are the
    // kernel's critical path).
    const int kq = tid & 3, prow = tid >> 2;
    int is_tile = 0, is_chunk = 0, is_slot = 0;  // next (tile, chunk) to fetch
    auto issue = [&]() {
      if (is_tile < my_tiles) {
        const int64_t r0 = static_cast<int64_t>(blockIdx.x + is_tile * gridDim.x) * kTileM + prow;
        const int k = is_chunk * kKC + kq * 4;
        const bool kin = k < p.K;
        const float* base = k < p.k1 ? p.A1 + k : p.A2 + (k - p.k1);
        const int64_t ld = k < p.k1 ? p.k1 : p.k2;
        const uint32_t slot = raw0 + is_slot * S::kRaw + tid * 16;
        if (p.scalar_a) {
          // rows not 16 B multiples (K = in + H with in % 4 != 0, or a narrow
          // A1 alone): element copies, each k from its own operand
#pragma unroll
          for (int it = 0; it < kRawPerThread; ++it) {
            const int64_t grow = r0 + kProducerRows * it;
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const int ke = k + e;
              const bool valid = ke < p.K && grow < p.M;
              const float* src = ke < p.k1 ? p.A1 + grow * p.k1 + ke : p.A2 + grow * p.k2 + (ke - p.k1);
              cp_async4_zfill(slot + it * kProducerThreads * 16 + 4 * e, valid ? src : p.A1, valid);
            }
          }
        } else {
#pragma unroll
          for (int it = 0; it < kRawPerThread; ++it) {
            const int64_t grow = r0 + kProducerRows * it;
            const bool valid = kin && grow < p.M;
            cp_async16_zfill(slot + it * kProducerThreads * 16, valid ? base + grow * ld : p.A1, valid);
          }
        }
        if (++is_chunk == p.nchunks) {
          is_chunk = 0;
          ++is_tile;
        }
        if (++is_slot == S::kRawSlots) is_slot = 0;
      }
      cp_async_commit();  // one group per item (possibly empty) keeps the accounting uniform
    };
    for (int i = 0; i < S::kRawSlots - 1; ++i) issue();
    int c = 0, slot_i = 0;
    uint32_t s = 0, ph = 0;
    for (int item = 0; item < total; ++item) {
      issue();
      cp_async_wait<S::kRawSlots - 1>();
      mbar_wait(&empty[s], ph ^ 1u);
      const uint32_t st = sbase + s * S::kStage;
      const uint8_t* slotp = smem + S::kRawOff + slot_i * S::kRaw + tid * 16;
      {
        // all four loads first, then split + store (exposes one LDS latency, not four)
        float4 v[kRawPerThread];
#pragma unroll
        for (int it = 0; it < kRawPerThread; ++it)
          v[it] = *reinterpret_cast<const float4*>(slotp + it * kProducerThreads * 16);
#pragma unroll
        for (int it = 0; it < kRawPerThread; ++it) {
          if (p.debug & 4) break;
          float h0, l0, h1, l1, h2, l2, h3, l3;
          split_tf32(v[it].x, h0, l0);
          split_tf32(v[it].y, h1, l1);
          split_tf32(v[it].z, h2, l2);
          split_tf32(v[it].w, h3, l3);
          const uint32_t off = tile_offset(kTileM, prow + kProducerRows * it, kq * 4);
          st_shared_v4(st + off, h0, h1, h2, h3);
          st_shared_v4(st + S::kA + off, l0, l1, l2, l3);
        }
        fence_async_smem();
        // every producer thread arrives (release of its own A stores); the
        // leader's arrival also arms the transaction count of the B copy
        if (tid == 0 && !(p.debug & 2)) {
          mbar_arrive_expect_tx(&full[s], 2 * S::kB);
          bulk_g2s(st + 2 * S::kA,
                   reinterpret_cast<const uint8_t*>(p.Bimg) + static_cast<int64_t>(c) * 2 * S::kB,
                   2 * S::kB, &full[s]);
        } else {
          mbar_arrive(&full[s]);
        }
      }
      if (++c == p.nchunks) c = 0;
      if (++slot_i == S::kRawSlots) slot_i = 0;
      if (++s == S::kStages) {
        s = 0;
        ph ^= 1u;
      }
    }
    cp_async_wait<0>();
  } else if (warp == kMmaWarp) {
    // ---------------- MMA issuer
    constexpr uint32_t idesc = idesc_tf32(kTileM, NPAD);
    constexpr uint32_t lboA = tile_lbo(kTileM), lboB = tile_lbo(NPAD);
    const int gs = (EPI == kEpiGru || EPI == kEpiGruBwd) ? p.gru_split : 0;
    const uint32_t idesc3 = gs ? idesc_tf32(kTileM, 3 * gs) : idesc;
    const uint32_t boffH = static_cast<uint32_t>(gs / 8) * 128u;  // B rows [H, 4H)
    uint32_t g = 0, it = 0;
    const bool split = (kEpiCell<EPI> || EPI == kEpiStore2) && p.split_acc;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
      const uint32_t b = split ? 0u : (it & 1u);
      mbar_wait(&tempty[b], (split ? (it & 1u) : ((it >> 1) & 1u)) ^ 1u);
      fence_after_sync();
      const uint32_t d = tmem + b * 256;
      for (int c = 0; c < p.nchunks; ++c, ++g) {
        const uint32_t s = g % S::kStages, ph = (g / S::kStages) & 1u;
        mbar_wait(&full[s], ph);
        fence_after_sync();
        const uint32_t st = sbase + s * S::kStage;
        if (lane == 0) {
          // GRU split: chunk 0 full N; X chunks N = 3H at column 0 ([n r z]);
          // Hm chunks N = 3H at column H ([r z hn])
          uint32_t id = idesc, dd = d, bo = 0;
          bool skip = false;
          if (gs && c > 0) {
            id = idesc3;
            if (c * kKC >= p.k1) {
              dd = d + static_cast<uint32_t>(gs);
              bo = boffH;
            }
          }
          if (EPI == kEpiStore2 && p.s2_gru && c * kKC >= 2 * p.s2_gru) {
            if (c * kKC >= 3 * p.s2_gru) {  // hn block -> h columns
              id = idesc_tf32(kTileM, p.s2_gru);
              dd = d + static_cast<uint32_t>(p.s2_h0);
              bo = static_cast<uint32_t>(p.s2_h0 / 8) * 128u;
            } else if (p.s2_nx > 0) {  // n block -> x columns
              id = idesc_tf32(kTileM, p.s2_nx);
            } else {
              skip = true;
            }
          }
#pragma unroll
          for (int ks = 0; ks < kKC / 8; ++ks) {
            if (skip) break;
            const uint64_t ahi = make_desc(st + 2 * ks * lboA, lboA, 128);
            const uint64_t alo = make_desc(st + S::kA + 2 * ks * lboA, lboA, 128);
            const uint64_t bhi = make_desc(st + 2 * S::kA + 2 * ks * lboB + bo, lboB, 128);
            const uint64_t blo = make_desc(st + 2 * S::kA + S::kB + 2 * ks * lboB + bo, lboB, 128);
            const uint32_t first = (c > 0 || ks > 0) ? 1u : 0u;
            mma_tf32(dd, ahi, bhi, id, first);
            const uint32_t dc = split ? dd + 256u : dd;
            mma_tf32(dc, ahi, blo, id, split ? first : 1u);
            mma_tf32(dc, alo, bhi, id, 1u);
          }
          commit(&empty[s]);
          if (c == p.nchunks - 1) commit(&tfull[b]);
        }
        __syncwarp();
      }
    }
  } else if (warp >= kEpiWarp0) {
    // ---------------- epilogue
    const int q = warp & 3, half = (warp - kEpiWarp0) >> 2;
    uint32_t it = 0;
    const bool split = (kEpiCell<EPI> || EPI == kEpiStore2) && p.split_acc;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
      const uint32_t b = split ? 0u : (it & 1u);
      const int64_t row0 = static_cast<int64_t>(tile) * kTileM + q * 32;  // this warp's 32 rows
      const int64_t row = row0 + lane;
      if (kEpiCell<EPI> && row < p.M) {
        // the per-row state operands do not depend on the MMAs: pull this
        // lane's segment of them into L1 while the tile's MMAs run (the
        // epilogue's global loads were its largest stall, ncu long_scoreboard)
        const int64_t off = row * p.H + half * (p.H / 2);
        auto pf = [](const float* ptr) {
          if (ptr) asm volatile("prefetch.global.L1 [%0];" ::"l"(ptr));
        };
        pf((EPI == kEpiLstm || EPI == kEpiLstmBwd) ? p.c_prev + off : p.h_skip + off);
        if (EPI == kEpiLstmBwd || EPI == kEpiGruBwd) {
          pf(p.dh + off);
          if (EPI == kEpiLstmBwd && p.dc) pf(p.dc + off);
        }
      }
      mbar_wait(&tfull[b], split ? (it & 1u) : ((it >> 1) & 1u));
      fence_after_sync();
      const uint32_t trow = tmem + b * 256 + (static_cast<uint32_t>(q * 32) << 16);
      // the four gate blocks of hidden units [j0, j0 + 16): hi*hi sums (+ the
      // correction sums when split)
      // H = 8: 8-column gate blocks (the first 8 entries of each array are
      // live, the rest are never stored)
      // (cell epilogues only: store2 leaves p.H unset)
      const bool narrow = kEpiCell<EPI> && NPAD == 64 && p.H < 16;  // 4H = 32: only the 64-column tile
      auto ld8_into = [&](uint32_t addr, float (&v)[16]) {
        float t[8];
        tmem_ld8(addr, t);
        tmem_wait_ld();
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = t[u];
#pragma unroll
        for (int u = 8; u < 16; ++u) v[u] = 0.f;
      };
      auto ld_gates = [&](int c0, int c1, int c2, int c3, float (&a0)[16], float (&a1)[16],
                          float (&a2)[16], float (&a3)[16]) {
        if (narrow) {
          ld8_into(trow + c0, a0);
          ld8_into(trow + c1, a1);
          ld8_into(trow + c2, a2);
          ld8_into(trow + c3, a3);
          if (split) {
            float t[16];
            ld8_into(trow + 256 + c0, t);
            for (int u = 0; u < 8; ++u) a0[u] += t[u];
            ld8_into(trow + 256 + c1, t);
            for (int u = 0; u < 8; ++u) a1[u] += t[u];
            ld8_into(trow + 256 + c2, t);
            for (int u = 0; u < 8; ++u) a2[u] += t[u];
            ld8_into(trow + 256 + c3, t);
            for (int u = 0; u < 8; ++u) a3[u] += t[u];
          }
          return;
        }
        tmem_ld16(trow + c0, a0);
        tmem_ld16(trow + c1, a1);
        tmem_ld16(trow + c2, a2);
        tmem_ld16(trow + c3, a3);
        tmem_wait_ld();
        if (split) {
          float t0[16], t1[16];
          tmem_ld16(trow + 256 + c0, t0);
          tmem_ld16(trow + 256 + c1, t1);
          tmem_wait_ld();
#pragma unroll
          for (int u = 0; u < 16; ++u) {
            a0[u] += t0[u];
            a1[u] += t1[u];
          }
          tmem_ld16(trow + 256 + c2, t0);
          tmem_ld16(trow + 256 + c3, t1);
          tmem_wait_ld();
#pragma unroll
          for (int u = 0; u < 16; ++u) {
            a2[u] += t0[u];
            a3[u] += t1[u];
          }
        }
      };
      // Coalesced store of a 32-row x 16-column register block (lane = row):
      // transposed through a per-warp smem buffer so each st.global.v4 covers
      // 8 rows x 64 contiguous bytes instead of 32 rows x 16 bytes.
      // 32 rows x 4 chunks of 16 B, chunk index XOR-swizzled by (row >> 1) & 3
      // so both the row-per-lane writes and the 8-rows-x-64B reads are
      // bank-conflict free.
      float* wb = reinterpret_cast<float*>(smem + S::kOut) + (warp - kEpiWarp0) * (32 * 16);
      auto stage_store = [&](const float (&v)[16], float* base, int64_t stride, int col0) {
        const int ncols = narrow ? 8 : 16;
#pragma unroll
        for (int u = 0; u < 16; u += 4)
          *reinterpret_cast<float4*>(wb + lane * 16 + (((u >> 2) ^ ((lane >> 1) & 3)) << 2)) =
              make_float4(v[u], v[u + 1], v[u + 2], v[u + 3]);
        __syncwarp();
        const int i = lane >> 2, k = lane & 3;
#pragma unroll
        for (int bb = 0; bb < 4; ++bb) {
          const int rl = bb * 8 + i;
          const float4 x = *reinterpret_cast<const float4*>(wb + rl * 16 + ((k ^ ((rl >> 1) & 3)) << 2));
          if (row0 + rl < p.M && k * 4 < ncols)
            *reinterpret_cast<float4*>(base + (row0 + rl) * stride + col0 + k * 4) = x;
        }
        __syncwarp();
      };
      auto load16 = [&](const float* base, int j0, float (&v)[16]) {
        if (base != nullptr && row < p.M) {
          const float* sp = base + row * p.H + j0;
#pragma unroll
          for (int u = 0; u < 16; u += 4) {
            float4 x = make_float4(0.f, 0.f, 0.f, 0.f);
            if (!narrow || u < 8) x = __ldg(reinterpret_cast<const float4*>(sp + u));
            v[u] = x.x; v[u + 1] = x.y; v[u + 2] = x.z; v[u + 3] = x.w;
          }
        } else {
#pragma unroll
          for (int u = 0; u < 16; ++u) v[u] = 0.f;
        }
      };
      // accumulator column block of each gate (GRU split: [n | r | z | hn])
      const bool gsplit = (EPI == kEpiGru || EPI == kEpiGruBwd) && p.gru_split;
      const int cb0 = gsplit ? p.H : 0, cb1 = gsplit ? 2 * p.H : p.H, cb2 = gsplit ? 0 : 2 * p.H;
      if (EPI == kEpiLstmBwd || EPI == kEpiGruBwd) {
        const int H = p.H;
        // hidden units of this warp: one half each (H >= 32), or all of them
        // in the first half (H = 16: one 16-column block)
        const bool small_h = NPAD == 64 && H < 32;  // compile-time false on the wide tiles
        const int jb = !small_h ? half * (H / 2) : (half ? H : 0);
        const int je = !small_h ? jb + H / 2 : H;
        for (int j0 = jb; j0 < je; j0 += 16) {
          float a0[16], a1[16], a2[16], a3[16];
          float cv[16];  // out: dc_prev (LSTM) / dh_skip (GRU)
          ld_gates(cb0 + j0, cb1 + j0, cb2 + j0, 3 * H + j0, a0, a1, a2, a3);
          // per-row operands 4 columns at a time (register budget of 152)
          const float* sp = (EPI == kEpiLstmBwd ? p.c_prev : p.h_skip) + row * H + j0;
          const float* dp = p.dh + row * H + j0;
          const float* cp = p.dc ? p.dc + row * H + j0 : nullptr;
#pragma unroll
          for (int u4 = 0; u4 < 16; u4 += 4) {
            float4 s4 = make_float4(0.f, 0.f, 0.f, 0.f), d4 = s4, c4 = s4;
            if (row < p.M && (!narrow || u4 < 8)) {
              s4 = __ldg(reinterpret_cast<const float4*>(sp + u4));
              d4 = __ldg(reinterpret_cast<const float4*>(dp + u4));
              if (EPI == kEpiLstmBwd && cp) c4 = __ldg(reinterpret_cast<const float4*>(cp + u4));
            }
            const float sv[4] = {s4.x, s4.y, s4.z, s4.w};
            const float dv[4] = {d4.x, d4.y, d4.z, d4.w};
            const float ci[4] = {c4.x, c4.y, c4.z, c4.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const int u = u4 + e;
              const int j = j0 + u;
              const float d = dv[e];
              if (EPI == kEpiLstmBwd) {
                const float ig = sigm(a0[u] + sbias[j]), fg = sigm(a1[u] + sbias[H + j]);
                const float gg = ftanh(a2[u] + sbias[2 * H + j]);
                const float og = sigm(a3[u] + sbias[3 * H + j]);
                const float tc = ftanh(fg * sv[e] + ig * gg);
                const float dct = (1.f - tc * tc) * (d * og) + ci[e];
                a0[u] = ig * (1.f - ig) * (dct * gg);
                a1[u] = fg * (1.f - fg) * (dct * sv[e]);
                a2[u] = (1.f - gg * gg) * (dct * ig);
                a3[u] = og * (1.f - og) * (d * tc);
                cv[u] = dct * fg;
              } else {
                const float rr = sigm(a0[u] + sbias[j]), zz = sigm(a1[u] + sbias[H + j]);
                const float hn = a3[u];
                const float nn = ftanh(a2[u] + rr * hn + sbias[2 * H + j]);
                const float dpre_n = (1.f - nn * nn) * (d * (1.f - zz));
                a0[u] = rr * (1.f - rr) * (dpre_n * hn);
                a1[u] = zz * (1.f - zz) * (d * (sv[e] - nn));
                a2[u] = dpre_n;
                a3[u] = dpre_n * rr;
                cv[u] = d * zz;
              }
            }
          }
          stage_store(a0, p.G, 4 * H, 0 * H + j0);
          stage_store(a1, p.G, 4 * H, 1 * H + j0);
          stage_store(a2, p.G, 4 * H, 2 * H + j0);
          stage_store(a3, p.G, 4 * H, 3 * H + j0);
          stage_store(cv, p.dstate, H, j0);
        }
      } else if (EPI == kEpiLstm || EPI == kEpiGru) {
        const int H = p.H;
        // hidden units of this warp: one half each (H >= 32), or all of them
        // in the first half (H = 16: one 16-column block)
        const bool small_h = NPAD == 64 && H < 32;  // compile-time false on the wide tiles
        const int jb = !small_h ? half * (H / 2) : (half ? H : 0);
        const int je = !small_h ? jb + H / 2 : H;
        for (int j0 = jb; j0 < je; j0 += 16) {
          float a0[16], a1[16], a2[16], a3[16];
          // state row prefetch overlaps the TMEM reads
          float sv[16];
          load16(EPI == kEpiLstm ? p.c_prev : p.h_skip, j0, sv);
          ld_gates(cb0 + j0, cb1 + j0, cb2 + j0, 3 * H + j0, a0, a1, a2, a3);
          if (!(p.debug & 1)) {
            float ho[16], co[16];
#pragma unroll
            for (int u = 0; u < 16; ++u) {
              const int j = j0 + u;
              const float p0 = a0[u] + sbias[j];
              const float p1 = a1[u] + sbias[H + j];
              if (EPI == kEpiLstm) {
                const float ig = sigm(p0), fg = sigm(p1);
                const float gg = ftanh(a2[u] + sbias[2 * H + j]);
                const float og = sigm(a3[u] + sbias[3 * H + j]);
                const float cc = fg * sv[u] + ig * gg;
                a0[u] = ig;
                a1[u] = fg;
                a2[u] = gg;
                a3[u] = og;
                co[u] = cc;
                ho[u] = og * ftanh(cc);
              } else {
                const float rr = sigm(p0), zz = sigm(p1);
                const float hn = a3[u];
                const float nn = ftanh(a2[u] + rr * hn + sbias[2 * H + j]);
                a0[u] = rr;
                a1[u] = zz;
                a2[u] = nn;
                ho[u] = (1.f - zz) * nn + zz * sv[u];
              }
            }
            if (p.gates != nullptr) {
              stage_store(a0, p.gates, 4 * H, 0 * H + j0);
              stage_store(a1, p.gates, 4 * H, 1 * H + j0);
              stage_store(a2, p.gates, 4 * H, 2 * H + j0);
              stage_store(a3, p.gates, 4 * H, 3 * H + j0);
            }
            if (EPI == kEpiLstm) stage_store(co, p.c_out, H, j0);
            stage_store(ho, p.h_out, H, j0);
          }
        }
      } else if (p.n1 % 16 == 0 && p.n2 % 16 == 0) {
        const int ncol = p.n1 + p.n2;
        for (int cb = half * 16; cb < ncol; cb += 32) {
          float a[16];
          tmem_ld16(trow + cb, a);
          tmem_wait_ld();
          if (split) {
            float t2[16];
            tmem_ld16(trow + 256 + cb, t2);
            tmem_wait_ld();
#pragma unroll
            for (int u = 0; u < 16; ++u) a[u] += t2[u];
          }
          if (cb < p.n1) {
            if (p.bias != nullptr) {
#pragma unroll
              for (int u = 0; u < 16; ++u) a[u] += sbias[cb + u];
            }
            if (p.store_accumulate && row < p.M) {
              const float* ep = p.C1 + row * p.n1 + cb;
#pragma unroll
              for (int u = 0; u < 16; u += 4) {
                const float4 e = *reinterpret_cast<const float4*>(ep + u);
                a[u] += e.x; a[u + 1] += e.y; a[u + 2] += e.z; a[u + 3] += e.w;
              }
            }
            if (p.relu) {
#pragma unroll
              for (int u = 0; u < 16; ++u) a[u] = a[u] > 0.f ? a[u] : 0.f;  // ref src/nn.cpp:19-25
            }
            stage_store(a, p.C1, p.n1, cb);
          } else {
            stage_store(a, p.C2, p.n2, cb - p.n1);
          }
        }
      } else {
        const int ncol = p.n1 + p.n2;
        const bool vec = p.n1 % 4 == 0 && p.n2 % 4 == 0 && p.bias == nullptr && !p.store_accumulate && !p.relu;
        for (int cb = half * 8; cb < ncol; cb += 16) {
          float a[8];
          tmem_ld8(trow + cb, a);
          tmem_wait_ld();
          if (split) {
            float t2[8];
            tmem_ld8(trow + 256 + cb, t2);
            tmem_wait_ld();
#pragma unroll
            for (int u = 0; u < 8; ++u) a[u] += t2[u];
          }
          if (row < p.M) {
            if (vec) {
#pragma unroll
              for (int u = 0; u < 8; u += 4) {
                const int col = cb + u;
                if (col < ncol) {
                  float* dst = col < p.n1 ? p.C1 + row * p.n1 + col : p.C2 + row * p.n2 + (col - p.n1);
                  *reinterpret_cast<float4*>(dst) = make_float4(a[u], a[u + 1], a[u + 2], a[u + 3]);
                }
              }
            } else {
              // narrow / odd widths (e.g. a prediction head with d = 2):
              // element stores with the bias / accumulate / ReLU epilogue
#pragma unroll
              for (int u = 0; u < 8; ++u) {
                const int col = cb + u;
                if (col >= ncol) continue;
                if (col < p.n1) {
                  float v = a[u];
                  if (p.bias != nullptr) v += sbias[col];
                  float* dst = p.C1 + row * p.n1 + col;
                  if (p.store_accumulate) v += *dst;
                  if (p.relu) v = v > 0.f ? v : 0.f;
                  *dst = v;
                } else {
                  p.C2[row * p.n2 + (col - p.n1)] = a[u];
                }
              }
            }
          }
        }
      }
      fence_before_sync();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[b]);
    }
  }
  __syncthreads();
  fence_after_sync();
  if (warp == kMmaWarp) tmem_free(tmem, 512);
}

// ------------------------------------------------------------- weight gradient
// Partial D'_cta (Mg x Npad) = sum over this CTA's rows of G^T(:, rows) *
// [X | Hm | 1](rows, :), with Mg = 4H in {128, 256} and Npad >= in + H + 1.
// Warps 0-15 copy raw 16-row chunks (cp.async, two chunks ahead) and write
// the transposed, 3xTF32-split operands; warp 16 issues the MMAs; warps 0-7
// drain the TMEM partial. Hand-offs
// are mbarriers only (no block-wide barrier per chunk): raw chunk landed
// (cp.async.mbarrier.arrive.noinc from every copier), raw slot consumed,
// operand stage full (every converter), stage free (tcgen05.commit).
// copy + convert threads: the conversion is issue-latency bound (ncu: "wait"
// and long-scoreboard stalls with 2 warps per scheduler at 256 threads)
constexpr int kWgConv = 512;
constexpr int kThreads = kWgConv + 32;     // + the MMA warp
constexpr int kKW = 16;  // rows (the MMA K) per staged chunk

template <int MG, int NPAD>
struct WgradSmem {
  static constexpr uint32_t kA = tile_bytes(MG, kKW);
  static constexpr uint32_t kB = tile_bytes(NPAD, kKW);
  static constexpr uint32_t kStage = 2 * kA + 2 * kB;
  static constexpr int kStages = 2;
  // raw fp32 chunk: G rows (MG) + X rows (<= 128) + Hm rows (<= 64), cp.async ring
  static constexpr int kRawSlots = 3;
  static constexpr uint32_t kRaw = kKW * 4 * (MG + 192);
  static constexpr uint32_t kRawOff = kStages * kStage;
  static constexpr uint32_t kBars = kRawOff + kRawSlots * kRaw;
  static constexpr uint32_t kBytes = kBars + 128;
};

__device__ __forceinline__ void cp_async_mbar_arrive_noinc(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}

template <int MG, int NPAD>
__global__ void __launch_bounds__(kThreads, 1)
k_wgrad(int M, int in, int H, const float* __restrict__ G, const float* __restrict__ X,
        const float* __restrict__ Hm, float* __restrict__ ws, int gw) {
  // gw: columns of G (<= MG; the rest of A' is zero — a linear layer with
  // fewer than 128 outputs)
  using S = WgradSmem<MG, NPAD>;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S::kBars);
  uint64_t* empty = full + S::kStages;
  uint64_t* rawfull = empty + S::kStages;
  uint64_t* rawempty = rawfull + S::kRawSlots;
  uint64_t* done = rawempty + S::kRawSlots;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  constexpr int kHalves = MG / 128;
  constexpr uint32_t kCols = kHalves == 2 ? 512 : 256;
  if (warp == 0) tmem_alloc(tmem_slot, kCols);
  if (tid == 0) {
    for (int s = 0; s < S::kStages; ++s) {
      mbar_init(&full[s], kWgConv);
      mbar_init(&empty[s], 1);
    }
    for (int r = 0; r < S::kRawSlots; ++r) {
      mbar_init(&rawfull[r], kWgConv);
      mbar_init(&rawempty[r], kWgConv);
    }
    mbar_init(done, 1);
    fence_barrier_init();
  }
  fence_before_sync();
  __syncthreads();
  fence_after_sync();
  const uint32_t tmem = *tmem_slot;
  const uint32_t sbase = smem_u32(smem);
  const int KXH = in + H;
  const int64_t per = (static_cast<int64_t>(M) + gridDim.x - 1) / gridDim.x;
  const int64_t rb = blockIdx.x * per;
  const int64_t re = rb + per < M ? rb + per : M;
  const int nchunks = re > rb ? static_cast<int>((re - rb + kKW - 1) / kKW) : 0;

  if (warp < kWgConv / 32) {
    // ---------------- copy + convert
    // raw slot layout: G [kKW][MG] | X [kKW][in] | Hm [kKW][H]
    const uint32_t raw0 = sbase + S::kRawOff;
    // The 16 rows of each operand are one contiguous block in global memory, so
    // each region is a linear copy; rows past `re` are zero-filled.
    auto copy_region = [&](uint32_t dst, const float* src, int width, int live_rows) {
      if (width % 4 != 0) {  // narrow operand (d = 2 input, a 2-wide head gradient): elements
        const int n1 = kKW * width, valid1 = live_rows * width;
        for (int f = tid; f < n1; f += kWgConv) {
          const bool valid = f < valid1;
          cp_async4_zfill(dst + f * 4, valid ? src + f : src, valid);
        }
        return;
      }
      const int n4 = kKW * width / 4, valid4 = live_rows * width / 4;
      for (int f = tid; f < n4; f += kWgConv) {
        const bool valid = f < valid4;
        cp_async16_zfill(dst + f * 16, valid ? src + f * 4 : src, valid);
      }
    };
    auto issue = [&](int c) {
      const int r = c % S::kRawSlots;
      if (c >= S::kRawSlots) mbar_wait(&rawempty[r], ((c - S::kRawSlots) / S::kRawSlots) & 1u);
      const uint32_t slot = raw0 + r * S::kRaw;
      const int64_t q0 = rb + static_cast<int64_t>(c) * kKW;
      const int live = static_cast<int>(re - q0 < kKW ? re - q0 : kKW);
      copy_region(slot, G + q0 * gw, gw, live);
      copy_region(slot + kKW * MG * 4, X + q0 * in, in, live);
      // Hm absent (a plain linear layer's weight gradient): zero columns
      copy_region(slot + kKW * (MG + in) * 4, Hm ? Hm + q0 * H : G, H, Hm ? live : 0);
      cp_async_mbar_arrive_noinc(&rawfull[r]);  // completes when every copier's copies landed
    };
    for (int c = 0; c < S::kRawSlots - 1 && c < nchunks; ++c) issue(c);
    for (int c = 0; c < nchunks; ++c) {
      if (c + S::kRawSlots - 1 < nchunks) issue(c + S::kRawSlots - 1);
      const int r = c % S::kRawSlots;
      mbar_wait(&rawfull[r], (c / S::kRawSlots) & 1u);
      const uint32_t s = c % S::kStages;
      if (c >= S::kStages) mbar_wait(&empty[s], ((c - S::kStages) / S::kStages) & 1u);
      const uint32_t st = sbase + s * S::kStage;
      const float* rawG = reinterpret_cast<const float*>(smem + S::kRawOff + r * S::kRaw);
      const float* rawX = rawG + kKW * MG;
      const float* rawH = rawX + kKW * in;
      const int64_t q0c = rb + static_cast<int64_t>(c) * kKW;
      // A' = G^T: one (column m, 4-row quad) per task; lanes take consecutive
      // columns so the 8 lanes of a store phase fill 8 distinct 16 B bank groups
      // of a core matrix (conflict-free), and the column reads are consecutive.
      for (int task = tid; task < MG * (kKW / 4); task += kWgConv) {
        const int m = task % MG, k4 = task / MG;
        float h[4], l[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) split_tf32(m < gw ? rawG[(k4 * 4 + q) * gw + m] : 0.f, h[q], l[q]);
        const uint32_t off = tile_offset(MG, m, k4 * 4);
        st_shared_v4(st + off, h[0], h[1], h[2], h[3]);
        st_shared_v4(st + S::kA + off, l[0], l[1], l[2], l[3]);
      }
      // B' = [X | Hm | 1]^T (ones column at n = in + H -> bias gradient)
      for (int task = tid; task < NPAD * (kKW / 4); task += kWgConv) {
        const int n = task % NPAD, k4 = task / NPAD;
        float h[4], l[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int rr = k4 * 4 + q;
          float x = 0.f;
          if (n < in) x = rawX[rr * in + n];
          else if (n < KXH) x = rawH[rr * H + (n - in)];
          else if (n == KXH && q0c + rr < re) x = 1.f;
          split_tf32(x, h[q], l[q]);
        }
        const uint32_t off = tile_offset(NPAD, n, k4 * 4);
        st_shared_v4(st + 2 * S::kA + off, h[0], h[1], h[2], h[3]);
        st_shared_v4(st + 2 * S::kA + S::kB + off, l[0], l[1], l[2], l[3]);
      }
      fence_async_smem();
      mbar_arrive(&full[s]);
      mbar_arrive(&rawempty[r]);
    }
  } else if (lane == 0) {
    // ---------------- MMA issuer (warp kWgConv / 32)
    constexpr uint32_t idesc = idesc_tf32(128, NPAD);
    constexpr uint32_t lboA = tile_lbo(MG), lboB = tile_lbo(NPAD);
    for (int c = 0; c < nchunks; ++c) {
      const uint32_t s = c % S::kStages;
      mbar_wait(&full[s], (c / S::kStages) & 1u);
      fence_after_sync();
      const uint32_t st = sbase + s * S::kStage;
#pragma unroll
      for (int ks = 0; ks < kKW / 8; ++ks) {
        const uint64_t bhi = make_desc(st + 2 * S::kA + 2 * ks * lboB, lboB, 128);
        const uint64_t blo = make_desc(st + 2 * S::kA + S::kB + 2 * ks * lboB, lboB, 128);
#pragma unroll
        for (int hf = 0; hf < kHalves; ++hf) {
          // rows [hf*128, hf*128+128) of A' start 16 core-matrix groups further
          const uint32_t aoff = hf * 16 * 128;
          const uint64_t ahi = make_desc(st + aoff + 2 * ks * lboA, lboA, 128);
          const uint64_t alo = make_desc(st + S::kA + aoff + 2 * ks * lboA, lboA, 128);
          const uint32_t d = tmem + hf * 256;
          mma_tf32(d, ahi, bhi, idesc, (c > 0 || ks > 0) ? 1u : 0u);
          mma_tf32(d, ahi, blo, idesc, 1u);
          mma_tf32(d, alo, bhi, idesc, 1u);
        }
      }
      commit(&empty[s]);
    }
    if (nchunks > 0) commit(done);
  }
  // ---------------- TMEM partial -> workspace (warps 0-7)
  if (warp < 8) {
    float* out = ws + static_cast<int64_t>(blockIdx.x) * MG * NPAD;
    if (nchunks > 0) {
      mbar_wait(done, 0);
      fence_after_sync();
    }
    const int q = warp & 3, half = warp >> 2;
    for (int hf = 0; hf < kHalves; ++hf) {
      const int m = hf * 128 + q * 32 + lane;
      const uint32_t trow = tmem + hf * 256 + (static_cast<uint32_t>(q * 32) << 16);
      for (int cb = half * 16; cb < NPAD; cb += 32) {
        float a[16];
        if (nchunks > 0) {
          tmem_ld16(trow + cb, a);
          tmem_wait_ld();
        } else {
#pragma unroll
          for (int u = 0; u < 16; ++u) a[u] = 0.f;
        }
#pragma unroll
        for (int u = 0; u < 16; u += 4)
          *reinterpret_cast<float4*>(out + static_cast<int64_t>(m) * NPAD + cb + u) =
              make_float4(a[u], a[u + 1], a[u + 2], a[u + 3]);
      }
    }
  }
  fence_before_sync();
  __syncthreads();
  fence_after_sync();
  if (warp == 0) tmem_free(tmem, kCols);
}

// dW[k][m] += sum_cta D'[cta][m][k] (k < in+H); db[m] += sum_cta D'[cta][m][in+H] (m < nb)
__global__ void k_wgrad_reduce(int nctas, int MG, int NPAD, int KXH, int wrows, int nb, int gw,
                               const float* __restrict__ ws, float* __restrict__ dW,
                               float* __restrict__ db) {
  const int64_t total = static_cast<int64_t>(gw) * (KXH + 1);
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int m = static_cast<int>(i / (KXH + 1));
    const int k = static_cast<int>(i % (KXH + 1));
    float acc = 0.f;
    for (int c = 0; c < nctas; ++c) acc += ws[(static_cast<int64_t>(c) * MG + m) * NPAD + k];
    if (k < KXH) {
      if (k < wrows) dW[static_cast<int64_t>(k) * gw + m] += acc;
    } else if (m < nb) {
      db[m] += acc;
    }
  }
}

int round_up(int x, int m) { return (x + m - 1) / m * m; }

template <int EPI, int NPAD>
void launch_row_gemm(const RowGemmArgs& a, cudaStream_t st) {
  const uint32_t smem = RowGemmSmem<NPAD>::kBytes;
  static bool configured = false;
  if (!configured) {
    DGNN_CUDA(cudaFuncSetAttribute(k_row_gemm<EPI, NPAD>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    configured = true;
  }
  const int ntiles = (a.M + kTileM - 1) / kTileM;
  // DGNN_GEMM_SMS caps the persistent grid (experiments: leaving SMs to a
  // concurrent SpMM on the other layer lane)
  static const int cap = [] {
    const char* e = std::getenv("DGNN_GEMM_SMS");
    const int v = e ? std::atoi(e) : kNumSMs;
    return v > 0 && v <= kNumSMs ? v : kNumSMs;
  }();
  const int grid = ntiles < cap ? ntiles : cap;
  DGNN_LAUNCH((k_row_gemm<EPI, NPAD>), grid, kRgThreads, smem, st, a);
}

template <int EPI>
void dispatch_row_gemm(int npad, const RowGemmArgs& a, cudaStream_t st) {
  switch (npad) {
    case 64: launch_row_gemm<EPI, 64>(a, st); break;
    case 128: launch_row_gemm<EPI, 128>(a, st); break;
    case 192: launch_row_gemm<EPI, 192>(a, st); break;
    case 256: launch_row_gemm<EPI, 256>(a, st); break;
    default: throw std::invalid_argument("umma row gemm: unsupported N " + std::to_string(npad));
  }
}

}  // namespace

bool umma_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("DGNN_DISABLE_UMMA");
    return !(e && e[0] == '1');
  }();
  return on;
}

bool umma_cell_supported(int in, int H) {
  // in + H <= 192: the weight-gradient kernel's raw [X | Hm] staging slot;
  // any in >= 1 (rows that are not 16 B multiples are copied by element);
  // H = 16 runs its 4H = 64 gate columns in the first epilogue half and pads
  // the weight gradient's row tile to 128; H = 8 works in 8-column blocks
  return umma_enabled() && (H == 8 || H == 16 || H == 32 || H == 64) && in >= 1 && in + H <= 192;
}

int umma_npad(int N) { return N <= 64 ? 64 : (N <= 128 ? 128 : (N <= 192 ? 192 : 256)); }

int64_t umma_bimage_floats(int N, int K) {
  const int npad = umma_npad(N);
  const int nchunks = (K + kKC - 1) / kKC;
  return static_cast<int64_t>(nchunks) * 2 * (tile_bytes(npad, kKC) / 4);
}

void umma_pack_b(const float* M, int ld, bool trans, int n0, int N, int K, float* out,
                 cudaStream_t stream) {
  const int npad = umma_npad(N);
  const int nchunks = (K + kKC - 1) / kKC;
  const int64_t total = static_cast<int64_t>(nchunks) * npad * kKC;
  DGNN_LAUNCH(k_pack_b, wave_grid(total, 256, 4), 256, 0, stream, M, ld, trans ? 1 : 0, n0, N, K,
              npad, nchunks, out, 0);
}

bool umma_gru_split(bool lstm, int in, int H) {
  static const bool on = [] {
    const char* e = std::getenv("DGNN_GRU_SPLIT");
    return !(e && e[0] == '0');
  }();
  return on && !lstm && in % kKC == 0 && H % 16 == 0 && umma_npad(4 * H) == 4 * H;
}

void umma_pack_cell_image(bool lstm, const float* W, int in, int H, float* out, cudaStream_t stream) {
  const int N = 4 * H, K = in + H;
  const int npad = umma_npad(N);
  const int nchunks = (K + kKC - 1) / kKC;
  const int64_t total = static_cast<int64_t>(nchunks) * npad * kKC;
  DGNN_LAUNCH(k_pack_b, wave_grid(total, 256, 4), 256, 0, stream, W, N, 1, 0, N, K, npad, nchunks,
              out, umma_gru_split(lstm, in, H) ? H : 0);
}

void umma_cell_forward(bool lstm, int n, int in, int H, const float* X, const float* Hm,
                       const float* h_skip, const float* c_prev, const float* Bimg,
                       const float* bias, float* gates, float* c, float* h, cudaStream_t stream) {
  RowGemmArgs a{};
  a.M = n;
  a.k1 = in;
  a.k2 = H;
  a.K = in + H;
  a.nchunks = (a.K + kKC - 1) / kKC;
  a.A1 = X;
  a.A2 = Hm;
  a.Bimg = Bimg;
  a.H = H;
  a.bias = bias;
  a.c_prev = c_prev;
  a.h_skip = h_skip;
  a.gates = gates;
  a.c_out = c;
  a.h_out = h;
  a.gru_split = umma_gru_split(lstm, in, H) ? H : 0;
  a.split_acc = umma_split_acc() & 1;
  a.scalar_a = in % 4 != 0;
  a.debug = umma_debug_flags();
  const int npad = umma_npad(4 * H);
  if (lstm) dispatch_row_gemm<kEpiLstm>(npad, a, stream);
  else dispatch_row_gemm<kEpiGru>(npad, a, stream);
}

void umma_cell_backward_recompute(bool lstm, int n, int in, int H, const float* X, const float* Hm,
                                  const float* h_skip, const float* c_prev, const float* Bimg,
                                  const float* bias, const float* dh, const float* dc, float* G,
                                  float* dstate, cudaStream_t stream) {
  RowGemmArgs a{};
  a.M = n;
  a.k1 = in;
  a.k2 = H;
  a.K = in + H;
  a.nchunks = (a.K + kKC - 1) / kKC;
  a.A1 = X;
  a.A2 = Hm;
  a.Bimg = Bimg;
  a.H = H;
  a.bias = bias;
  a.c_prev = c_prev;
  a.h_skip = h_skip;
  a.dh = dh;
  a.dc = dc;
  a.G = G;
  a.dstate = dstate;
  a.gru_split = umma_gru_split(lstm, in, H) ? H : 0;
  a.split_acc = (umma_split_acc() >> 1) & 1;
  a.scalar_a = in % 4 != 0;
  a.debug = umma_debug_flags();
  const int npad = umma_npad(4 * H);
  if (lstm) dispatch_row_gemm<kEpiLstmBwd>(npad, a, stream);
  else dispatch_row_gemm<kEpiGruBwd>(npad, a, stream);
}

void umma_gemm_store2(int n, int K, const float* A, const float* Bimg, int n1, int n2, float* C1,
                      float* C2, cudaStream_t stream, const float* bias, bool accumulate, int gru_h,
                      bool relu, bool split_acc) {
  if (n1 > 256) throw std::invalid_argument("umma_gemm_store2: at most 256 bias columns");
  RowGemmArgs a{};
  a.split_acc = split_acc && (umma_split_acc() & 1);
  a.scalar_a = K % 4 != 0;
  a.bias = bias;
  a.relu = relu ? 1 : 0;
  a.store_accumulate = accumulate ? 1 : 0;
  a.M = n;
  a.k1 = K;
  a.k2 = 0;
  a.K = K;
  a.nchunks = (K + kKC - 1) / kKC;
  a.A1 = A;
  a.A2 = A;
  a.Bimg = Bimg;
  a.n1 = n1;
  a.n2 = n2;
  a.C1 = C1;
  a.C2 = C2;
  // GRU: K = 4H gate columns [r z n hn]; C1 | C2 = [dX | dHm] (n1 = in,
  // n2 = H) or dHm alone (n1 = H, n2 = 0)
  if (gru_h > 0 && K == 4 * gru_h && umma_gru_split(false, kKC, gru_h) && n1 % 16 == 0) {
    a.s2_gru = gru_h;
    a.s2_nx = n2 > 0 ? n1 : 0;
    a.s2_h0 = n2 > 0 ? n1 : 0;
  }
  a.debug = umma_debug_flags();
  dispatch_row_gemm<kEpiStore2>(umma_npad(n1 + n2), a, stream);
}

// CTAs of the weight gradient for n rows: >= ~128 rows each (every CTA writes
// a 4H x Npad partial the reduction reads back) and <= kWgRowsPerCta rows
// each. The tensor core adds into its fp32 accumulator with truncation, so
// the error of one CTA's partial grows with the rows it sums; capping them
// bounds it (1M rows / 148 CTAs measured 4.8e-5 norm-relative vs fp64) and
// the fixed-order reduction of the partials is exact-rounded fp32.
constexpr int64_t kWgRowsPerCta = 8192;
int wgrad_grid(int64_t n) {
  const int64_t cap = (n + kWgRowsPerCta - 1) / kWgRowsPerCta;
  if (cap > kNumSMs) return static_cast<int>((cap + kNumSMs - 1) / kNumSMs * kNumSMs);
  return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(kNumSMs, n / 128)));
}

int64_t umma_wgrad_workspace(int64_t n, int in, int H) {
  const int need = round_up(in + H + 1, 16);
  const int npad = need <= 144 ? 144 : (need <= 208 ? 208 : 256);
  const int mg = H == 64 ? 256 : 128;  // the kernel's row tile (4H padded up to 128)
  return static_cast<int64_t>(wgrad_grid(n)) * mg * npad;
}

void umma_wgrad(int n, int in, int H, const float* G, const float* X, const float* Hm, float* dW,
                int nb, float* db, float* ws, cudaStream_t stream, int gw) {
  if (gw <= 0) gw = 4 * H;
  if (gw > 4 * H) throw std::invalid_argument("umma_wgrad: G wider than 4H");
  if (n <= 0) return;  // no rows: nothing to accumulate
  const int need = round_up(in + H + 1, 16);
  const int npad = need <= 144 ? 144 : (need <= 208 ? 208 : 256);
  const int grid = wgrad_grid(n);
  if (umma_wgrad_mn_supported(in, H, gw, G, X, Hm)) {
    // TMA-fed MN-major kernel (umma_wgrad.cu)
    const int np = umma_wgrad_mn(n, in, H, G, gw, X, Hm, ws, grid, stream);
    const int kxh = in + (Hm ? H : 0);
    const int64_t total = static_cast<int64_t>(gw) * (kxh + 1);
    DGNN_LAUNCH(k_wgrad_reduce, wave_grid(total, 256, 4), 256, 0, stream, grid, 4 * H, np, kxh, kxh, nb, gw, ws,
                dW, db);
    return;
  }
  auto go = [&](auto mg_tag, auto np_tag) {
    constexpr int MG = decltype(mg_tag)::value, NP = decltype(np_tag)::value;
    const uint32_t smem = WgradSmem<MG, NP>::kBytes;
    static bool configured = false;
    if (!configured) {
      DGNN_CUDA(cudaFuncSetAttribute(k_wgrad<MG, NP>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      configured = true;
    }
    DGNN_LAUNCH((k_wgrad<MG, NP>), grid, kThreads, smem, stream, n, in, H, G, X, Hm, ws, gw);
  };
  if (H == 64) {
    if (npad == 144) go(std::integral_constant<int, 256>{}, std::integral_constant<int, 144>{});
    else if (npad == 208) go(std::integral_constant<int, 256>{}, std::integral_constant<int, 208>{});
    else go(std::integral_constant<int, 256>{}, std::integral_constant<int, 256>{});
  } else {
    if (npad == 144) go(std::integral_constant<int, 128>{}, std::integral_constant<int, 144>{});
    else if (npad == 208) go(std::integral_constant<int, 128>{}, std::integral_constant<int, 208>{});
    else go(std::integral_constant<int, 128>{}, std::integral_constant<int, 256>{});
  }
  const int64_t total = static_cast<int64_t>(gw) * (in + H + 1);
  DGNN_LAUNCH(k_wgrad_reduce, wave_grid(total, 256, 4), 256, 0, stream, grid, H == 64 ? 256 : 128, npad, in + H,
              Hm ? in + H : in, nb, gw, ws, dW, db);
}

}  // namespace cuda
}  // namespace dgnn
