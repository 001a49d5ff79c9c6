// K4 gather of sampled feature rows and K6 argmax assignment.
//
//   csc_gather_rows : feats.rows[sampling.indices]   (pipeline.py:176, sampling.py:52-54)
//   csc_assign      : assign(soft)                   (sampling.py:197-220)
#include <algorithm>
#include <cmath>

#include "internal.cuh"

namespace csc {
namespace {

template <typename T>
__global__ void k_gather(const T* __restrict__ F, int64_t ldf, int ncols, const int64_t* __restrict__ idx, int64_t n,
                         int64_t N, T* __restrict__ out, int64_t ldo, int* __restrict__ bad) {
  const int64_t total = n * ncols;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = t / ncols;
    const int c = (int)(t - i * ncols);
    const int64_t r = idx[i];
    if (r < 0 || r >= N) {
      atomicOr(bad, 1);
      continue;
    }
    out[i * ldo + c] = F[r * ldf + c];
  }
}

// per-block column sums of squares of a row-major N x k block
template <typename T>
__global__ void k_colsq_rows(const T* __restrict__ A, int64_t ld, int64_t n, int k, double* __restrict__ part) {
  const int64_t rows_per_block = (n + gridDim.x - 1) / gridDim.x;
  const int64_t r0 = blockIdx.x * rows_per_block;
  const int64_t r1 = min(n, r0 + rows_per_block);
  for (int c = threadIdx.x; c < k; c += blockDim.x) {
    double s = 0.0;
    for (int64_t r = r0; r < r1; ++r) {
      const double v = (double)A[r * ld + c];
      s += v * v;
    }
    part[(size_t)blockIdx.x * k + c] = s;
  }
}

__global__ void k_colnorm(const double* __restrict__ part, int nblocks, int k, double* __restrict__ norm,
                          int* __restrict__ any_nonzero) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < k; c += gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int b = 0; b < nblocks; ++b) s += part[(size_t)b * k + c];
    norm[c] = sqrt(s);
    if (norm[c] > 0.0) atomicOr(any_nonzero, 1);
  }
}

// warp per row: argmax of soft/||col|| with lowest-index ties; zero-norm columns
// never win; identically-zero rows take the raw argmax (index 0) and are flagged.
template <typename T>
__global__ void k_argmax(const T* __restrict__ A, int64_t ld, int64_t n, int k, const double* __restrict__ norm,
                         int64_t* __restrict__ labels, uint8_t* __restrict__ fallback,
                         unsigned long long* __restrict__ nfb) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = warp; r < n; r += nw) {
    double best = -INFINITY;
    int bidx = -1;
    bool nonzero = false;
    for (int c = lane; c < k; c += 32) {
      const double v = (double)A[r * ld + c];
      nonzero |= v != 0.0;
      const double nc = norm[c];
      const double q = nc > 0.0 ? v / nc : -INFINITY;
      if (bidx < 0 || q > best) {  // strict '>': lowest column wins ties within the lane
        best = q;
        bidx = c;
      }
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, best, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bidx, o);
      const bool take = oi >= 0 && (bidx < 0 || ob > best || (ob == best && oi < bidx));
      if (take) {
        best = ob;
        bidx = oi;
      }
    }
    const bool any = __any_sync(0xffffffffu, nonzero);
    if (lane == 0) {
      labels[r] = any ? bidx : 0;
      if (fallback) fallback[r] = any ? 0 : 1;
      if (!any) atomicAdd(nfb, 1ull);
    }
  }
}

// column-sharded variant: per-row (best value, global column, any nonzero)
template <typename T>
__global__ void k_argmax_partial(const T* __restrict__ A, int64_t ld, int64_t n, int k, const double* __restrict__ norm,
                                 int64_t col_offset, double* __restrict__ bval, int64_t* __restrict__ bcol,
                                 uint8_t* __restrict__ nz) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = warp; r < n; r += nw) {
    double best = -INFINITY;
    int bidx = -1;
    bool nonzero = false;
    for (int c = lane; c < k; c += 32) {
      const double v = (double)A[r * ld + c];
      nonzero |= v != 0.0;
      const double q = norm[c] > 0.0 ? v / norm[c] : -INFINITY;
      if (bidx < 0 || q > best) {
        best = q;
        bidx = c;
      }
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, best, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bidx, o);
      if (oi >= 0 && (bidx < 0 || ob > best || (ob == best && oi < bidx))) {
        best = ob;
        bidx = oi;
      }
    }
    const bool any = __any_sync(0xffffffffu, nonzero);
    if (lane == 0) {
      bval[r] = best;
      bcol[r] = col_offset + bidx;
      nz[r] = any ? 1 : 0;
    }
  }
}

template <typename T>
void assign_partial_typed(const T* A, int64_t ld, int64_t n, int k, int device, int64_t col_offset, double* bval,
                          int64_t* bcol, uint8_t* nz, int* any_norm, cudaStream_t s) {
  const int nb = (int)std::max<int64_t>(1, std::min<int64_t>(n, (int64_t)device_props(device).sms * 4));
  Scratch part(sizeof(double) * (size_t)nb * k, s), norm(sizeof(double) * k, s), flag(sizeof(int), s);
  CSC_CUDA(cudaMemsetAsync(flag.get(), 0, sizeof(int), s));
  k_colsq_rows<T><<<nb, 256, 0, s>>>(A, ld, n, k, part.as<double>());
  CSC_LAUNCHED();
  k_colnorm<<<(k + 127) / 128, 128, 0, s>>>(part.as<double>(), nb, k, norm.as<double>(), flag.as<int>());
  CSC_LAUNCHED();
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((n + 7) / 8, (int64_t)device_props(device).sms * 16));
  k_argmax_partial<T><<<grid, 256, 0, s>>>(A, ld, n, k, norm.as<double>(), col_offset, bval, bcol, nz);
  CSC_LAUNCHED();
  CSC_CUDA(cudaMemcpyAsync(any_norm, flag.get(), sizeof(int), cudaMemcpyDeviceToHost, s));
}

template <typename T>
void assign_typed(const T* A, int64_t ld, int64_t n, int k, int device, int64_t* labels, uint8_t* fb,
                  unsigned long long* nfb, cudaStream_t s) {
  const int nb = (int)std::max<int64_t>(1, std::min<int64_t>(n, (int64_t)device_props(device).sms * 4));
  Scratch part(sizeof(double) * (size_t)nb * k, s), norm(sizeof(double) * k, s), flag(sizeof(int), s);
  CSC_CUDA(cudaMemsetAsync(flag.get(), 0, sizeof(int), s));
  k_colsq_rows<T><<<nb, 256, 0, s>>>(A, ld, n, k, part.as<double>());
  CSC_LAUNCHED();
  k_colnorm<<<(k + 127) / 128, 128, 0, s>>>(part.as<double>(), nb, k, norm.as<double>(), flag.as<int>());
  CSC_LAUNCHED();
  int any = 0;
  CSC_CUDA(cudaMemcpyAsync(&any, flag.get(), sizeof(int), cudaMemcpyDeviceToHost, s));
  CSC_CUDA(cudaStreamSynchronize(s));
  if (!any) fail(CSC_ERR_INVALID, "all indicator vectors are zero");
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((n + 7) / 8, (int64_t)device_props(device).sms * 16));
  k_argmax<T><<<grid, 256, 0, s>>>(A, ld, n, k, norm.as<double>(), labels, fb, nfb);
  CSC_LAUNCHED();
}

}  // namespace
}  // namespace csc

using namespace csc;

extern "C" {

int csc_gather_rows(const void* F, int64_t ldf, int64_t num_rows, int ncols, int io_dtype, const int64_t* idx,
                    int64_t n, void* out, int64_t ldo, int device, void* stream) {
  return guard([&] {
    if (ncols < 0 || n < 0 || num_rows < 0) fail(CSC_ERR_INVALID, "negative size");
    if (ldf < ncols || ldo < ncols) fail(CSC_ERR_INVALID, "leading dimension smaller than ncols");
    const size_t es = dtype_size(io_dtype);
    if (n == 0 || ncols == 0) return;
    if (!F || !idx || !out) fail(CSC_ERR_INVALID, "NULL buffer");
    DeviceGuard dg(device);
    ensure_pool(device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    DeviceView dF(F, es * (size_t)std::max<int64_t>(num_rows * ldf, 1), device, s);
    DeviceView didx(idx, sizeof(int64_t) * n, device, s);
    const bool odev = is_device_ptr(out, device);
    Scratch ob;
    void* dst = out;
    int64_t ld = ldo;
    if (!odev) {
      ob.alloc(es * n * ncols, s);
      dst = ob.get();
      ld = ncols;
    }
    Scratch bad(sizeof(int), s);
    CSC_CUDA(cudaMemsetAsync(bad.get(), 0, sizeof(int), s));
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((n * ncols + 255) / 256, 4096));
    if (io_dtype == CSC_F64)
      k_gather<double><<<grid, 256, 0, s>>>(dF.as<double>(), ldf, ncols, didx.as<int64_t>(), n, num_rows,
                                            static_cast<double*>(dst), ld, bad.as<int>());
    else
      k_gather<float><<<grid, 256, 0, s>>>(dF.as<float>(), ldf, ncols, didx.as<int64_t>(), n, num_rows,
                                           static_cast<float*>(dst), ld, bad.as<int>());
    CSC_LAUNCHED();
    if (!odev) copy_rows(out, ldo, dst, ncols, n, ncols, es, cudaMemcpyDeviceToHost, s);
    int hb = 0;
    CSC_CUDA(cudaMemcpyAsync(&hb, bad.get(), sizeof(int), cudaMemcpyDeviceToHost, s));
    CSC_CUDA(cudaStreamSynchronize(s));
    if (hb) fail(CSC_ERR_INVALID, "row index out of range");
  });
}

int csc_assign(const void* soft, int64_t ld, int64_t num_rows, int k, int io_dtype, int64_t* labels,
               uint8_t* fallback, int64_t* num_fallback, int device, void* stream) {
  return guard([&] {
    if (k < 1 || num_rows < 0 || ld < k) fail(CSC_ERR_INVALID, "soft indicators must be (N, k)");
    const size_t es = dtype_size(io_dtype);
    if (num_rows == 0) fail(CSC_ERR_INVALID, "all indicator vectors are zero");
    if (!soft || !labels) fail(CSC_ERR_INVALID, "NULL buffer");
    DeviceGuard dg(device);
    ensure_pool(device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    DeviceView dA(soft, es * (size_t)num_rows * ld, device, s);
    DeviceOut lab(labels, sizeof(int64_t) * num_rows, device, s);
    DeviceOut fb(fallback, (size_t)num_rows, device, s);
    Scratch nfb(sizeof(unsigned long long), s);
    CSC_CUDA(cudaMemsetAsync(nfb.get(), 0, sizeof(unsigned long long), s));
    if (io_dtype == CSC_F64)
      assign_typed<double>(dA.as<double>(), ld, num_rows, k, device, lab.as<int64_t>(), fb.as<uint8_t>(),
                           nfb.as<unsigned long long>(), s);
    else
      assign_typed<float>(dA.as<float>(), ld, num_rows, k, device, lab.as<int64_t>(), fb.as<uint8_t>(),
                          nfb.as<unsigned long long>(), s);
    lab.finish();
    fb.finish();
    unsigned long long h = 0;
    CSC_CUDA(cudaMemcpyAsync(&h, nfb.get(), sizeof(h), cudaMemcpyDeviceToHost, s));
    CSC_CUDA(cudaStreamSynchronize(s));
    if (num_fallback) *num_fallback = (int64_t)h;
  });
}

int csc_assign_partial(const void* soft, int64_t ld, int64_t num_rows, int k, int io_dtype, int64_t col_offset,
                       double* best_val, int64_t* best_col, uint8_t* nonzero, int* any_norm, int device,
                       void* stream) {
  return guard([&] {
    if (k < 1 || num_rows < 0 || ld < k) fail(CSC_ERR_INVALID, "soft indicators must be (N, k)");
    if (col_offset < 0) fail(CSC_ERR_INVALID, "col_offset must be >= 0");
    const size_t es = dtype_size(io_dtype);
    if (num_rows == 0) {
      if (any_norm) *any_norm = 0;
      return;
    }
    if (!soft || !best_val || !best_col || !nonzero) fail(CSC_ERR_INVALID, "NULL buffer");
    DeviceGuard dg(device);
    ensure_pool(device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    DeviceView dA(soft, es * (size_t)num_rows * ld, device, s);
    DeviceOut bv(best_val, sizeof(double) * num_rows, device, s);
    DeviceOut bc(best_col, sizeof(int64_t) * num_rows, device, s);
    DeviceOut nzo(nonzero, (size_t)num_rows, device, s);
    int h_any = 0;
    if (io_dtype == CSC_F64)
      assign_partial_typed<double>(dA.as<double>(), ld, num_rows, k, device, col_offset, bv.as<double>(),
                                   bc.as<int64_t>(), nzo.as<uint8_t>(), &h_any, s);
    else
      assign_partial_typed<float>(dA.as<float>(), ld, num_rows, k, device, col_offset, bv.as<double>(),
                                  bc.as<int64_t>(), nzo.as<uint8_t>(), &h_any, s);
    bv.finish();
    bc.finish();
    nzo.finish();
    CSC_CUDA(cudaStreamSynchronize(s));
    if (any_norm) *any_norm = h_any;
  });
}

}  // extern "C"
