// Host launchers for the dense kernels (dense_kernels.cu): the fused
// GraphRNN cell (K4/K5/K6), linear layers (K7/K8), MAE (K9), Adam (K10).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace dgnn {
namespace cuda {

// Fused cell forward (ref cell_core_forward, src/cells.cpp:102-132).
// W: (in+H) x 4H row-major combined gate weights, bias: 4H (see pack_cell).
// gates (n x 4H) receives LSTM i,f,g,o / GRU r,z,n,hn (the CellTape); LSTM
// writes c; both write h. X: n x in, Hm: n x H, h_skip (GRU), c_prev (LSTM).
void cell_forward(bool lstm, int n, int in, int H, const float* X, const float* Hm,
                  const float* h_skip, const float* c_prev, const float* W, const float* bias,
                  float* gates, float* c, float* h, cudaStream_t stream);

// Pointwise half of cell_core_backward (src/cells.cpp:134-195): writes the
// gate-gradient matrix G (n x 4H: LSTM dpre_i,f,g,o / GRU dpre_r,z,n,d_hn) and
// dc_prev (LSTM) or dh_skip (GRU).
void cell_backward_pointwise(bool lstm, int n, int H, const float* gates, const float* c,
                             const float* c_prev, const float* h_skip, const float* dh,
                             const float* dc, float* G, float* dc_prev, float* dh_skip,
                             cudaStream_t stream);

// C = [A1 | A2] * B (+ bias) (relu) with C written as [C1 | C2] column blocks,
// or accumulated (C += ...) when `accumulate`. A1: m x k1, A2: m x k2 (may be
// null, k2 = 0), B: (k1+k2) x (n1+n2) with row stride ldb, C1: m x n1,
// C2: m x n2 (may be null).
void gemm_nn(int m, int k1, int k2, int n1, int n2, const float* A1, const float* A2,
             const float* B, int ldb, const float* bias, bool relu, bool accumulate, float* C1,
             float* C2, cudaStream_t stream);

// dpre = (out > 0) ? dout : 0 (relu backward, ref src/nn.cpp:33-34).
void relu_backward(int64_t n, const float* out, const float* dout, float* dpre,
                   cudaStream_t stream);

// D (k1+k2) x nc += [A1 | A2]^T * B over m rows with a fixed-order split over
// m (deterministic). bias_grad (nb entries, may be null) += column sums of the
// first nb columns of B. `ws` must hold gemm_tn_workspace(...) floats.
int64_t gemm_tn_workspace(int m, int k, int nc);
void gemm_tn_acc(int m, int k1, int k2, int nc, const float* A1, const float* A2, const float* B,
                 float* D, int nb, float* bias_grad, float* ws, cudaStream_t stream);

// out (cols x rows) = in (rows x cols)^T.
void transpose(int rows, int cols, const float* in, float* out, cudaStream_t stream);

// y += alpha * x (n elements).
void axpy(int64_t n, float alpha, const float* x, float* y, cudaStream_t stream);

// MAE over seed rows [r0, r1) (ref loss_mae src/nn.cpp:62-71, seed_loss
// src/train.cpp:119-144). dpred (n x d) is fully written: sign(diff)/(rows*d)
// * inv_h on seed rows, 0 elsewhere. loss_out (double) += value * inv_h.
void mae_loss(int n, int d, int r0, int r1, const float* pred, const float* target,
              float* dpred, double inv_h, double* loss_out, double* ws, cudaStream_t stream);

// flag = 1 if any of x[0..n) is not finite.
void nonfinite_check(int64_t n, const float* x, int32_t* flag, cudaStream_t stream);

// Adam / SGD (ref optimizer_step src/train.cpp:26-52). Skips entirely when
// *skip_flag != 0. grad is pre-scaled by `gscale`.
void adam_step(int64_t n, float* p, float* m, float* v, const float* g, float gscale, float lr,
               float beta1, float beta2, float eps, float bc1, float bc2, bool sgd,
               const int32_t* skip_flag, cudaStream_t stream);

// Reference flat cell layout [wx_g (in x H), uh_g (H x H), b_g (H)]_g  <->
// combined W ((in+H) x 4H) and bias (4H). GRU: blocks r,z,xn,hn with the
// xn block zero on the Hm rows and the hn block zero on the X rows.
void pack_cell(bool lstm, int in, int H, const float* flat, float* W, float* bias,
               cudaStream_t stream);
// flat_grad += unpack(dW, db).
// Per-cell weight / bias gradient accumulators of a model, for the batched
// zeroing and unpacking below (one launch per sample for all cells).
struct CellGradDesc {
  float* dW;
  float* db;
  int lstm, in, H;
  int64_t offset;  // the cell's first parameter in the flat buffer
};
void zero_cell_grads(const CellGradDesc* cells_dev, int n, int64_t max_elems, cudaStream_t stream);
void unpack_cell_grads(const CellGradDesc* cells_dev, int n, int64_t max_elems, float* flat_grad,
                       cudaStream_t stream);

void unpack_cell_grad(bool lstm, int in, int H, const float* dW, const float* db,
                      float* flat_grad, cudaStream_t stream);

}  // namespace cuda
}  // namespace dgnn
