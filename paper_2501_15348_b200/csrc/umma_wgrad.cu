// Weight gradient of the cell / linear layers on tcgen05 with MN-major
// operands fed by TMA (ref src/cells.cpp:167-195, the
// wx / uh / b accumulations of cell_core_backward, and src/nn.cpp linear
// gradients):
//
//   D'(4H x Npad) = sum over rows of G^T(:, row) * [X | Hm | 1](row, :)
//
// The reduction dimension is the row dimension, so both operands are read
// "MN-major": a 16-row chunk of G (row-major, n x gw) is already the K x M
// tile the tensor core wants, and likewise X and Hm. The TMA engine copies
// each chunk straight from the row-major activations into MN-major
// 128 B-swizzled, 32 B-granule atoms (box = 32 columns x 16 rows); the tensor
// core reads those raw fp32 tiles as the TF32 "hi" operand (top 19 bits, i.e.
// trunc_tf32), and converter warps write only the "lo" = x - trunc(x) tiles,
// elementwise at the same swizzled offsets — no transposition, no per-element
// shuffling through registers. 3xTF32: hi*hi + hi*lo + lo*hi.
//
//   warps 0-7  converters (lo tiles), then drain TMEM to the CTA's partial
//   warp 8     TMA producer (one elected lane)
//   warp 9     TMEM allocation + the MMA issuer (one lane)
//
// A stage holds raw + lo tiles of A' (gw/32 atoms of G, zero atoms up to 4H)
// and B' (X atoms, Hm atoms, one constant atom holding the ones column that
// yields the bias gradient); full (TMA bytes) -> lo_ready (converters) ->
// empty (tcgen05.commit) mbarriers hand a stage around. Every CTA sums a
// chunk-aligned row range; partials are reduced in fixed order
// (k_wgrad_reduce), so the result is deterministic.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <stdexcept>
#include <string>
#include <type_traits>

#include "common.cuh"
#include "umma.cuh"
#include "umma_kernels.h"

namespace dgnn {
namespace cuda {
namespace {

using namespace umma;

constexpr int kChunkRows = 16;     // rows (the MMA K) per stage
constexpr int kAtomCols = 32;      // fp32 columns per 128 B swizzle atom
constexpr uint32_t kAtomBytes = kChunkRows * 128;  // one TMA box: 16 rows x 128 B
constexpr int kConvWarps = 8;
constexpr int kProdWarp = kConvWarps;
constexpr int kMmaWarp = kConvWarps + 1;
constexpr int kThreadsMn = 32 * (kConvWarps + 2);

template <int MG, int NPAD>
struct MnSmem {
  static constexpr int kAAtoms = MG / kAtomCols;
  static constexpr int kBAtoms = (NPAD + kAtomCols - 1) / kAtomCols;
  static constexpr uint32_t kA = kAAtoms * kAtomBytes;
  static constexpr uint32_t kB = kBAtoms * kAtomBytes;
  static constexpr uint32_t kStage = 2 * kA + 2 * kB;  // A raw | A lo | B raw | B lo
  static constexpr int kStages = (200 * 1024) / kStage < 6 ? (200 * 1024) / kStage : 6;
  static constexpr uint32_t kBars = kStages * kStage;
  static constexpr uint32_t kBytes = kBars + 256 + 1024;  // + alignment slack
  static_assert(kStages >= 2, "weight-gradient stage does not fit");
};

// SM100 smem descriptor for MN-major TF32 operands. The only MN-major layout
// the tensor core takes for 32-bit elements is "128 B swizzle, 32 B atom"
// (layout type 1, SWIZZLE_128B_BASE32B; cf. CUTLASS sm100_common.inl "for
// mn-major tf32 operands, SW128_32B is the only available smem layout"):
// Swizzle<2,5,2> on byte addresses — the four 32 B granules of a 128 B row
// are permuted by (row % 4) — over the canonical ((8,n),(4,k)) in 16 B units:
// 128 B of M/N per row, K rows 128 B apart, 4-row groups SBO = 512 B apart,
// 32-column blocks LBO apart (ref cute::UMMA::make_umma_desc<Major::MN>).
// The TMA engine writes exactly this with CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B.
__device__ __forceinline__ uint64_t make_desc_mn32(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFFu);
  d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFFu) << 16;
  d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFFu) << 32;
  d |= static_cast<uint64_t>(1) << 46;
  d |= static_cast<uint64_t>(1) << 61;
  return d;
}

// kind::tf32, fp32 accumulate, A and B MN-major
__host__ __device__ constexpr uint32_t idesc_tf32_mn(int M, int N) {
  return (1u << 4) | (2u << 7) | (2u << 10) | (1u << 15) | (1u << 16) |
         (static_cast<uint32_t>(N >> 3) << 17) | (static_cast<uint32_t>(M >> 4) << 24);
}

__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, int x, int y,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ float4 lo_of(float4 v) {
  auto lo = [](float x) { return x - __uint_as_float(__float_as_uint(x) & 0xFFFFE000u); };
  return make_float4(lo(v.x), lo(v.y), lo(v.z), lo(v.w));
}

// gw: G columns (multiple of 32, <= MG); xa / ha: X / Hm atoms (ha = 0 for a
// linear layer); ones column at KXH = 32 * (xa + ha) (the first column of
// atom xa + ha).
template <int MG, int NPAD>
__global__ void __launch_bounds__(kThreadsMn, 1)
k_wgrad_mn(const __grid_constant__ CUtensorMap tmG, const __grid_constant__ CUtensorMap tmX,
           const __grid_constant__ CUtensorMap tmH, int64_t M, int gw, int xa, int ha,
           int64_t chunks_per_cta, float* __restrict__ ws) {
  using S = MnSmem<MG, NPAD>;
  extern __shared__ uint8_t smem_raw[];
  // 1024 B alignment for the swizzle atoms
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S::kBars);
  uint64_t* lo_ready = full + S::kStages;
  uint64_t* empty = lo_ready + S::kStages;
  uint64_t* done = empty + S::kStages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  constexpr int kHalves = MG / 128;
  constexpr uint32_t kCols = kHalves == 2 ? 512 : 256;
  const int ga = gw / kAtomCols;
  const int ones_atom = xa + ha;

  const int64_t total_chunks = (M + kChunkRows - 1) / kChunkRows;
  const int64_t c0 = static_cast<int64_t>(blockIdx.x) * chunks_per_cta;
  const int64_t c1 = std::min<int64_t>(c0 + chunks_per_cta, total_chunks);
  const int nchunks = c1 > c0 ? static_cast<int>(c1 - c0) : 0;

  if (warp == kMmaWarp) tmem_alloc(tmem_slot, kCols);
  if (tid == 0) {
    for (int s = 0; s < S::kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&lo_ready[s], 32 * kConvWarps);
      mbar_init(&empty[s], 1);
    }
    mbar_init(done, 1);
    fence_barrier_init();
  }
  // constant atoms of every stage: zero G atoms past gw, the ones column
  // (raw) / zeros (lo), zero B atoms past the ones atom
  for (int s = 0; s < S::kStages; ++s) {
    uint8_t* st = smem + s * S::kStage;
    for (int a = ga; a < S::kAAtoms; ++a)
      for (int i = tid; i < static_cast<int>(kAtomBytes / 16); i += kThreadsMn) {
        reinterpret_cast<float4*>(st + a * kAtomBytes)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
        reinterpret_cast<float4*>(st + S::kA + a * kAtomBytes)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
      }
    for (int a = ones_atom; a < S::kBAtoms; ++a)
      for (int i = tid; i < static_cast<int>(kAtomBytes / 16); i += kThreadsMn) {
        const int r = i / 8, chunk = i % 8;  // row, physical 16 B chunk
        // column 0 of row r: logical 32 B granule 0 sits at granule r % 4
        const float one = (a == ones_atom && chunk == 2 * (r % 4)) ? 1.f : 0.f;
        reinterpret_cast<float4*>(st + 2 * S::kA + a * kAtomBytes)[i] = make_float4(one, 0.f, 0.f, 0.f);
        reinterpret_cast<float4*>(st + 2 * S::kA + S::kB + a * kAtomBytes)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
      }
  }
  fence_async_smem();
  fence_before_sync();
  __syncthreads();
  fence_after_sync();
  const uint32_t tmem = *tmem_slot;
  const uint32_t sbase = smem_u32(smem);

  if (warp == kProdWarp) {
    if (lane == 0) {
      const uint32_t bytes = static_cast<uint32_t>(ga + xa + ha) * kAtomBytes;
      for (int c = 0; c < nchunks; ++c) {
        const int s = c % S::kStages;
        if (c >= S::kStages) mbar_wait(&empty[s], ((c / S::kStages) - 1) & 1u);
        const uint32_t st = sbase + s * S::kStage;
        const int row = static_cast<int>((c0 + c) * kChunkRows);
        mbar_arrive_expect_tx(&full[s], bytes);
        for (int a = 0; a < ga; ++a) tma_load_2d(st + a * kAtomBytes, &tmG, a * kAtomCols, row, &full[s]);
        for (int a = 0; a < xa; ++a)
          tma_load_2d(st + 2 * S::kA + a * kAtomBytes, &tmX, a * kAtomCols, row, &full[s]);
        for (int a = 0; a < ha; ++a)
          tma_load_2d(st + 2 * S::kA + (xa + a) * kAtomBytes, &tmH, a * kAtomCols, row, &full[s]);
      }
    }
  } else if (warp == kMmaWarp) {
    if (lane == 0) {
      constexpr uint32_t idesc = idesc_tf32_mn(128, NPAD);
      for (int c = 0; c < nchunks; ++c) {
        const int s = c % S::kStages;
        mbar_wait(&lo_ready[s], (c / S::kStages) & 1u);
        fence_after_sync();
        const uint32_t st = sbase + s * S::kStage;
#pragma unroll
        for (int ks = 0; ks < kChunkRows / 8; ++ks) {
          const uint32_t koff = ks * 1024u;  // rows 8ks..8ks+7 of the chunk
          const uint64_t bhi = make_desc_mn32(st + 2 * S::kA + koff, kAtomBytes, 512);
          const uint64_t blo = make_desc_mn32(st + 2 * S::kA + S::kB + koff, kAtomBytes, 512);
#pragma unroll
          for (int hf = 0; hf < kHalves; ++hf) {
            const uint32_t aoff = hf * 4 * kAtomBytes + koff;  // gate rows 128 hf .. (4 atoms)
            const uint64_t ahi = make_desc_mn32(st + aoff, kAtomBytes, 512);
            const uint64_t alo = make_desc_mn32(st + S::kA + aoff, kAtomBytes, 512);
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
  } else {
    // ---------------- converters: lo tiles at the raw tiles' swizzled offsets
    constexpr int kThr = 32 * kConvWarps;
    const int na4 = ga * static_cast<int>(kAtomBytes / 16);
    const int nb4 = (xa + ha) * static_cast<int>(kAtomBytes / 16);
    for (int c = 0; c < nchunks; ++c) {
      const int s = c % S::kStages;
      mbar_wait(&full[s], (c / S::kStages) & 1u);
      uint8_t* st = smem + s * S::kStage;
      const float4* ar = reinterpret_cast<const float4*>(st);
      float4* al = reinterpret_cast<float4*>(st + S::kA);
      const float4* br = reinterpret_cast<const float4*>(st + 2 * S::kA);
      float4* bl = reinterpret_cast<float4*>(st + 2 * S::kA + S::kB);
      for (int i = tid; i < na4; i += kThr) al[i] = lo_of(ar[i]);
      for (int i = tid; i < nb4; i += kThr) bl[i] = lo_of(br[i]);
      fence_async_smem();
      mbar_arrive(&lo_ready[s]);
    }
  }
  // ---------------- TMEM partial -> workspace (warps 0-7)
  if (warp < kConvWarps) {
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
  if (warp == kMmaWarp) tmem_free(tmem, kCols);
}

// -------------------------------------------------------------- host side
using EncodeTiled = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                 const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                 CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiled encode_fn() {
  static EncodeTiled fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    DGNN_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    if (p == nullptr || q != cudaDriverEntryPointSuccess)
      throw std::runtime_error("cuTensorMapEncodeTiled unavailable");
    return reinterpret_cast<EncodeTiled>(p);
  }();
  return fn;
}

// row-major rows x cols fp32 matrix, boxes of 32 columns x 16 rows, 128 B
// swizzle with 32 B granules (the MN-major TF32 operand layout)
CUtensorMap make_map(const float* base, int64_t rows, int cols) {
  CUtensorMap m;
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(cols) * 4};
  const cuuint32_t box[2] = {kAtomCols, kChunkRows};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides,
                                 box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw std::runtime_error("cuTensorMapEncodeTiled failed: " + std::to_string(r));
  return m;
}

bool mn_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("DGNN_WGRAD_MN");
    return !(e && e[0] == '0');
  }();
  return on;
}

}  // namespace

bool umma_wgrad_mn_supported(int in, int H, int gw, const float* G, const float* X, const float* Hm) {
  auto al = [](const void* p) { return p == nullptr || reinterpret_cast<uintptr_t>(p) % 16 == 0; };
  const int hw = Hm ? H : 0;
  return mn_enabled() && (H == 32 || H == 64) && gw % kAtomCols == 0 && gw <= 4 * H && in % kAtomCols == 0 &&
         hw % kAtomCols == 0 && in + hw + 16 <= 256 && al(G) && al(X) && al(Hm);
}

int umma_wgrad_mn_npad(int in, int H, bool has_hm) {
  const int kxh = in + (has_hm ? H : 0);
  return kxh + 16 <= 144 ? 144 : (kxh + 16 <= 208 ? 208 : 256);
}

// D' partials of `grid` CTAs into ws (grid x 4H x npad); returns npad.
int umma_wgrad_mn(int64_t n, int in, int H, const float* G, int gw, const float* X, const float* Hm,
                  float* ws, int grid, cudaStream_t stream) {
  const int npad = umma_wgrad_mn_npad(in, H, Hm != nullptr);
  const CUtensorMap tg = make_map(G, n, gw);
  const CUtensorMap tx = make_map(X, n, in);
  const CUtensorMap th = Hm ? make_map(Hm, n, H) : tx;
  const int64_t total_chunks = (n + kChunkRows - 1) / kChunkRows;
  const int64_t per = (total_chunks + grid - 1) / grid;
  const int xa = in / kAtomCols, ha = Hm ? H / kAtomCols : 0;
  auto go = [&](auto mg_tag, auto np_tag) {
    constexpr int MG = decltype(mg_tag)::value, NP = decltype(np_tag)::value;
    const uint32_t smem = MnSmem<MG, NP>::kBytes;
    static bool configured = false;
    if (!configured) {
      DGNN_CUDA(cudaFuncSetAttribute(k_wgrad_mn<MG, NP>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      configured = true;
    }
    DGNN_LAUNCH((k_wgrad_mn<MG, NP>), grid, kThreadsMn, smem, stream, tg, tx, th, n, gw, xa, ha, per, ws);
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
  return npad;
}

}  // namespace cuda
}  // namespace dgnn
