// Stochastic block model edges on the device, bit-identical to the reference generator
// (sbm.py:83-100 _success_positions, sbm.py:118-155 sbm_generate).
//
// The reference walks the k(k+1)/2 community pairs (a <= b) in order; pair t has
// `cells` candidate node pairs, each an edge with probability q (q1 inside a community,
// q2 across), and draws batches of rng.geometric(q, size=batch) gaps until the running
// position passes `cells`; positions below `cells` are edges (diagonal pairs unpack a
// lower-triangle index, off-diagonal ones a row-major index).  For q < 1/3 numpy's
// geometric is ceil(-E / log1p(-q)) with E one standard-exponential draw, so the whole
// graph is one stream of exponential draws cut into per-pair segments:
//   1. E_0 .. E_{D-1} from the seeded PCG64 stream (numpy_exponentials, npzig.cu);
//   2. per-draw pair id (segment starts + scan); gap = ceil(-E / log1p(-q_pair));
//   3. position = -1 + segmented inclusive scan of the gaps;
//   4. every pair must end at or past its cells (else the reference draws another
//      batch: the host grows that pair's draw count and the pass repeats);
//   5. keep positions < cells, map them to (src, dst) in draw order.
// Pairs with q >= 1/3 use numpy's search method and are left to the host generator.
#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>

#include <cmath>
#include <vector>

#include "internal.cuh"

namespace csc {
namespace {

__global__ void k_seg_starts(const int64_t* __restrict__ doff, int64_t npairs, int32_t* __restrict__ flag) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x + 1; t < npairs; t += (int64_t)gridDim.x * blockDim.x)
    flag[doff[t]] = 1;  // draw counts are >= 1, so segment starts are distinct
}

__global__ void k_gaps(const double* __restrict__ E, const int32_t* __restrict__ seg, const double* __restrict__ l1mq,
                       int64_t D, int64_t* __restrict__ gap) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < D; i += (int64_t)gridDim.x * blockDim.x) {
    const double z = ceil(__ddiv_rn(-E[i], l1mq[seg[i]]));  // random_geometric_inversion
    gap[i] = z >= 9.223372036854776e18 ? INT64_MAX : (int64_t)z;
  }
}

__global__ void k_pair_last(const int64_t* __restrict__ csum, const int64_t* __restrict__ doff, int64_t npairs,
                            int64_t* __restrict__ last) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < npairs; t += (int64_t)gridDim.x * blockDim.x)
    last[t] = csum[doff[t + 1] - 1] - 1;
}

__global__ void k_keep(const int64_t* __restrict__ csum, const int32_t* __restrict__ seg,
                       const int64_t* __restrict__ cells, int64_t D, uint8_t* __restrict__ keep) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < D; i += (int64_t)gridDim.x * blockDim.x)
    keep[i] = (csum[i] - 1) < cells[seg[i]] ? 1 : 0;
}

// sbm.py _unpack_lower: t = i(i-1)/2 + j, 0 <= j < i
__device__ inline void unpack_lower(int64_t t, int64_t& i, int64_t& j) {
  const double r = __dadd_rn(1.0, sqrt(__dadd_rn(1.0, __dmul_rn(8.0, (double)t))));
  i = (int64_t)__ddiv_rn(r, 2.0);
  if (i * (i - 1) / 2 > t) i -= 1;
  if (i * (i - 1) / 2 + i <= t) i += 1;
  j = t - i * (i - 1) / 2;
}

__global__ void k_edges(const int64_t* __restrict__ kept, const int64_t* __restrict__ nkept,
                        const int64_t* __restrict__ csum, const int32_t* __restrict__ seg,
                        const int32_t* __restrict__ diag, const int64_t* __restrict__ rfirst,
                        const int64_t* __restrict__ cfirst, const int64_t* __restrict__ csize, int64_t* __restrict__ src,
                        int64_t* __restrict__ dst) {
  const int64_t E = *nkept;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < E; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = kept[e];
    const int32_t t = seg[i];
    const int64_t p = csum[i] - 1;
    if (diag[t]) {
      int64_t a, b;
      unpack_lower(p, a, b);
      src[e] = rfirst[t] + a;
      dst[e] = rfirst[t] + b;
    } else {
      src[e] = rfirst[t] + p / csize[t];
      dst[e] = cfirst[t] + p % csize[t];
    }
  }
}

inline int grid_for(int64_t n) { return (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 16)); }

}  // namespace
}  // namespace csc

using namespace csc;

extern "C" int csc_sbm_edges(uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo, int64_t npairs,
                             const int64_t* cells, const double* log1m_q, const int64_t* batch, const int32_t* diag,
                             const int64_t* row_first, const int64_t* col_first, const int64_t* col_size,
                             int64_t capacity, int64_t* src, int64_t* dst, int64_t* num_edges, int64_t* raw_consumed,
                             int device, void* stream) {
  return guard([&] {
    if (npairs < 0 || capacity < 0) fail(CSC_ERR_INVALID, "sbm: negative size");
    if (!num_edges) fail(CSC_ERR_INVALID, "sbm: num_edges is NULL");
    if (npairs > INT32_MAX) fail(CSC_ERR_INVALID, "sbm: too many community pairs");
    if (npairs > 0 && (!cells || !log1m_q || !batch || !diag || !row_first || !col_first || !col_size))
      fail(CSC_ERR_INVALID, "sbm: NULL pair array");
    for (int64_t t = 0; t < npairs; ++t) {
      if (cells[t] <= 0 || batch[t] <= 0) fail(CSC_ERR_INVALID, "sbm: pairs must have cells > 0 and batch > 0");
      if (!(log1m_q[t] < 0.0) || !(log1m_q[t] > std::log1p(-1.0 / 3.0)))
        fail(CSC_ERR_INVALID, "sbm: pair probability outside (0, 1/3) (numpy's inversion branch)");
      if (!diag[t] && col_size[t] <= 0) fail(CSC_ERR_INVALID, "sbm: off-diagonal pair with empty column block");
    }
    *num_edges = 0;
    if (raw_consumed) *raw_consumed = 0;
    if (npairs == 0) return;
    DeviceGuard dg(device);
    ensure_pool(device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const size_t pb = sizeof(int64_t) * npairs;
    DeviceView dCells(cells, pb, device, s), dL(log1m_q, sizeof(double) * npairs, device, s),
        dDiag(diag, sizeof(int32_t) * npairs, device, s), dRf(row_first, pb, device, s),
        dCf(col_first, pb, device, s), dCs(col_size, pb, device, s);
    std::vector<int64_t> nb(npairs, 1);  // batches per pair
    for (int round = 0; round < 64; ++round) {
      std::vector<int64_t> doff(npairs + 1, 0);
      for (int64_t t = 0; t < npairs; ++t) doff[t + 1] = doff[t] + batch[t] * nb[t];
      const int64_t D = doff[npairs];
      if (D > INT32_MAX * 8ll) fail(CSC_ERR_INVALID, "sbm: draw stream too long");
      Scratch E(sizeof(double) * D, s), segf(sizeof(int32_t) * D, s), seg(sizeof(int32_t) * D, s),
          gap(sizeof(int64_t) * D, s), csum(sizeof(int64_t) * D, s), ddoff(sizeof(int64_t) * (npairs + 1), s),
          last(pb, s);
      const int64_t raws = numpy_exponentials(state_hi, state_lo, inc_hi, inc_lo, D, E.as<double>(), s);
      CSC_CUDA(cudaMemcpyAsync(ddoff.get(), doff.data(), sizeof(int64_t) * (npairs + 1), cudaMemcpyHostToDevice, s));
      CSC_CUDA(cudaMemsetAsync(segf.get(), 0, sizeof(int32_t) * D, s));
      k_seg_starts<<<grid_for(npairs), 256, 0, s>>>(ddoff.as<int64_t>(), npairs, segf.as<int32_t>());
      CSC_LAUNCHED();
      size_t tb = 0;
      CSC_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tb, segf.as<int32_t>(), seg.as<int32_t>(), D, s));
      {
        Scratch tmp(tb, s);
        CSC_CUDA(cub::DeviceScan::InclusiveSum(tmp.get(), tb, segf.as<int32_t>(), seg.as<int32_t>(), D, s));
        CSC_LAUNCHED();
      }
      k_gaps<<<grid_for(D), 256, 0, s>>>(E.as<double>(), seg.as<int32_t>(), dL.as<double>(), D, gap.as<int64_t>());
      CSC_LAUNCHED();
      tb = 0;
      CSC_CUDA(cub::DeviceScan::InclusiveSumByKey(nullptr, tb, seg.as<int32_t>(), gap.as<int64_t>(),
                                                  csum.as<int64_t>(), D, cub::Equality(), s));
      {
        Scratch tmp(tb, s);
        CSC_CUDA(cub::DeviceScan::InclusiveSumByKey(tmp.get(), tb, seg.as<int32_t>(), gap.as<int64_t>(),
                                                    csum.as<int64_t>(), D, cub::Equality(), s));
        CSC_LAUNCHED();
      }
      k_pair_last<<<grid_for(npairs), 256, 0, s>>>(csum.as<int64_t>(), ddoff.as<int64_t>(), npairs,
                                                   last.as<int64_t>());
      CSC_LAUNCHED();
      std::vector<int64_t> hlast(npairs);
      CSC_CUDA(cudaMemcpyAsync(hlast.data(), last.get(), pb, cudaMemcpyDeviceToHost, s));
      CSC_CUDA(cudaStreamSynchronize(s));
      // the reference keeps drawing batches while last < cells; the first pair that
      // needs another batch shifts every later segment, so grow it and redo the pass
      bool short_pair = false;
      for (int64_t t = 0; t < npairs; ++t)
        if (hlast[t] < cells[t]) {
          ++nb[t];
          short_pair = true;
          break;
        }
      if (short_pair) continue;
      Scratch keep(D, s), kept(sizeof(int64_t) * D, s), nkept(sizeof(int64_t), s);
      k_keep<<<grid_for(D), 256, 0, s>>>(csum.as<int64_t>(), seg.as<int32_t>(), dCells.as<int64_t>(), D,
                                         keep.as<uint8_t>());
      CSC_LAUNCHED();
      tb = 0;
      thrust::counting_iterator<int64_t> it(0);
      CSC_CUDA(cub::DeviceSelect::Flagged(nullptr, tb, it, keep.as<uint8_t>(), kept.as<int64_t>(), nkept.as<int64_t>(),
                                          D, s));
      {
        Scratch tmp(tb, s);
        CSC_CUDA(cub::DeviceSelect::Flagged(tmp.get(), tb, it, keep.as<uint8_t>(), kept.as<int64_t>(),
                                            nkept.as<int64_t>(), D, s));
        CSC_LAUNCHED();
      }
      int64_t E_count = 0;
      CSC_CUDA(cudaMemcpyAsync(&E_count, nkept.get(), sizeof(int64_t), cudaMemcpyDeviceToHost, s));
      CSC_CUDA(cudaStreamSynchronize(s));
      *num_edges = E_count;
      if (raw_consumed) *raw_consumed = raws;
      if (E_count > capacity) fail(CSC_ERR_INVALID, "sbm: edge capacity too small (need *num_edges)");
      if (E_count == 0) return;
      if (!src || !dst) fail(CSC_ERR_INVALID, "sbm: NULL edge output");
      DeviceOut os(src, sizeof(int64_t) * E_count, device, s), od(dst, sizeof(int64_t) * E_count, device, s);
      k_edges<<<grid_for(E_count), 256, 0, s>>>(kept.as<int64_t>(), nkept.as<int64_t>(), csum.as<int64_t>(),
                                                seg.as<int32_t>(), dDiag.as<int32_t>(), dRf.as<int64_t>(),
                                                dCf.as<int64_t>(), dCs.as<int64_t>(), os.as<int64_t>(),
                                                od.as<int64_t>());
      CSC_LAUNCHED();
      os.finish();
      od.finish();
      CSC_CUDA(cudaStreamSynchronize(s));
      return;
    }
    fail(CSC_ERR_INVALID, "sbm: batch growth did not converge");
  });
}
