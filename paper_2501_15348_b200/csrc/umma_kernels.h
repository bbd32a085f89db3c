// tcgen05 3xTF32 kernels for the GraphRNN cell (umma_kernels.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace dgnn {
namespace cuda {

// Shapes the tensor-core path covers (others use the FFMA kernels).
bool umma_cell_supported(int in, int H);
// Process-wide switch (env DGNN_DISABLE_UMMA=1 forces the FFMA path).
bool umma_enabled();

int umma_npad(int N);
// floats of a packed B image for an N x K operand
int64_t umma_bimage_floats(int N, int K);
// Packed B image: B(n, k) = trans ? M[k*ld + n0+n] : M[(n0+n)*ld + k], split
// into TF32 hi/lo tiles in the canonical UMMA layout, K chunked by 32.
// Forward-contraction B image of a packed cell weight W ((in+H) x 4H): W^T,
// GRU gate columns permuted when umma_gru_split (used by umma_cell_forward /
// umma_cell_backward_recompute, which must be given this image).
bool umma_gru_split(bool lstm, int in, int H);
void umma_pack_cell_image(bool lstm, const float* W, int in, int H, float* out, cudaStream_t stream);
void umma_pack_b(const float* M, int ld, bool trans, int n0, int N, int K, float* out,
                 cudaStream_t stream);

// Fused cell forward: [X | Hm] * W (+ bias) -> gates / c / h (as cell_forward).
void umma_cell_forward(bool lstm, int n, int in, int H, const float* X, const float* Hm,
                       const float* h_skip, const float* c_prev, const float* Bimg,
                       const float* bias, float* gates, float* c, float* h, cudaStream_t stream);

// Gate recompute + pointwise cell backward (no gates tape): the same
// contraction as umma_cell_forward, epilogue writes G (n x 4H, the gate
// pre-activation gradients) and dstate = dc_prev (LSTM) / dh_skip (GRU).
// dc may be null (zero upstream cell gradient).
void umma_cell_backward_recompute(bool lstm, int n, int in, int H, const float* X, const float* Hm,
                                  const float* h_skip, const float* c_prev, const float* Bimg,
                                  const float* bias, const float* dh, const float* dc, float* G,
                                  float* dstate, cudaStream_t stream);

// [C1 | C2] = A (n x K) * B^T with B the packed (n1+n2) x K image; with
// `bias` (n1 entries) C1 gets + bias, with `accumulate` C1 += the product
// (both need 16-column blocks).
void umma_gemm_store2(int n, int K, const float* A, const float* Bimg, int n1, int n2, float* C1,
                      float* C2, cudaStream_t stream, const float* bias = nullptr,
                      bool accumulate = false, int gru_h = 0, bool relu = false,
                      bool split_acc = false);

// dW ((in+H) x 4H) += [X|Hm]^T G, db (nb) += colsum(G[:, :nb]); deterministic.
// Hm == nullptr: a plain linear layer's gradient, dW (in x gw) += X^T G with
// G n x gw, gw <= 4H (default 4H; H then only sizes the tile: 4H in {128, 256}).
int64_t umma_wgrad_workspace(int64_t n, int in, int H);
// TMA-fed MN-major variant (umma_wgrad.cu): shapes it covers, and the
// partials of `grid` CTAs into ws (returns the partial's column pitch)
bool umma_wgrad_mn_supported(int in, int H, int gw, const float* G, const float* X, const float* Hm);
int umma_wgrad_mn_npad(int in, int H, bool has_hm);
int umma_wgrad_mn(int64_t n, int in, int H, const float* G, int gw, const float* X, const float* Hm,
                  float* ws, int grid, cudaStream_t stream);
void umma_wgrad(int n, int in, int H, const float* G, const float* X, const float* Hm, float* dW,
                int nb, float* db, float* ws, cudaStream_t stream, int gw = 0);

}  // namespace cuda
}  // namespace dgnn
