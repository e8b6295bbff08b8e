// Collectives among mesh devices co-located on one GPU (and the relayouts
// around NCCL calls in the multi-process mode).  Semantics follow the
// reference's group operations exactly (spmd_interp.py:74-123):
//
//   gather-style  all_slice (:76-81), all_gather (:82-91), all_to_all
//                 (:105-122): pure data movement, bit-exact.  Written as a
//                 gather so every output store is coalesced:
//                 out[d][l] = src[table[d][combo(l)]][base[d] + sum (l_k % ext_k) * sstride_k]
//   reduce-style  all_reduce (:92-97), reduce_scatter (:98-104): the left fold
//                 of `_combine` (:66-71) in group (device) order, so the fp32
//                 result is bit-identical to the reference's np.add chain.
#include "common.cuh"

namespace {

__global__ void __launch_bounds__(256) gather_kernel(const __grid_constant__ spx_gather_params p) {
  SPX_PDL_ENTRY();
  const int d = blockIdx.y;
  const float* const* table = reinterpret_cast<const float* const*>(p.src_table);
  const int64_t* base = reinterpret_cast<const int64_t*>(p.base_off);
  float* out = reinterpret_cast<float* const*>(p.dst)[d];
  const int64_t b = base[d];
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < p.numel;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t rem = e, combo = 0, soff = b;
#pragma unroll
    for (int k = SPX_MAX_RANK - 1; k >= 0; --k) {
      if (k >= p.rank) continue;
      const int64_t lk = (k == 0) ? rem : rem % p.dims[k];
      rem = (k == 0) ? 0 : rem / p.dims[k];
      const int64_t q = lk / p.ext[k], r = lk - q * p.ext[k];
      combo += q * p.cmul[k];
      soff += r * p.sstride[k];
    }
    out[e] = table[(int64_t)d * p.n_combo + combo][soff];
  }
}

// Contiguous-source fast path: rank-1 copy of a chunk (all_slice of a dim-0
// chunk, dim-0 all_gather pieces) with float4 moves.
__global__ void __launch_bounds__(256) creduce_kernel(const __grid_constant__ spx_creduce_params p) {
  SPX_PDL_ENTRY();
  const int d = blockIdx.y;
  const float* const* src = reinterpret_cast<const float* const*>(p.src);
  const int32_t* mem = reinterpret_cast<const int32_t*>(p.members) + (int64_t)d * p.n_members;
  const int64_t b = reinterpret_cast<const int64_t*>(p.base_off)[d];
  float* out = reinterpret_cast<float* const*>(p.dst)[d];
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < p.numel;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t rem = e, soff = b;
#pragma unroll
    for (int k = SPX_MAX_RANK - 1; k >= 0; --k) {
      if (k >= p.rank) continue;
      const int64_t lk = (k == 0) ? rem : rem % p.dims[k];
      rem = (k == 0) ? 0 : rem / p.dims[k];
      soff += lk * p.sstride[k];
    }
    float acc = src[mem[0]][soff];
    for (int j = 1; j < p.n_members; ++j) {
      const float v = src[mem[j]][soff];
      acc = p.monoid == 0 ? f_add(acc, v) : f_max(acc, v);
    }
    out[e] = acc;
  }
}

// Contiguous rank-1 fold (the copy-engine reduce-scatter's member chunks):
// float4 per thread, all members' loads in flight before the fold.
__global__ void __launch_bounds__(256) creduce_vec_kernel(const __grid_constant__ spx_creduce_params p) {
  SPX_PDL_ENTRY();
  const int d = blockIdx.y;
  const float* const* src = reinterpret_cast<const float* const*>(p.src);
  const int32_t* mem = reinterpret_cast<const int32_t*>(p.members) + (int64_t)d * p.n_members;
  const int64_t b = reinterpret_cast<const int64_t*>(p.base_off)[d];
  float4* out = reinterpret_cast<float4*>(reinterpret_cast<float* const*>(p.dst)[d]);
  const int64_t n4 = p.numel >> 2;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
    float4 v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j)
      if (j < p.n_members) v[j] = reinterpret_cast<const float4*>(src[mem[j]] + b)[i];
    float4 acc = v[0];
#pragma unroll
    for (int j = 1; j < 8; ++j) {
      if (j >= p.n_members) break;
      if (p.monoid == 0) {
        acc.x = f_add(acc.x, v[j].x); acc.y = f_add(acc.y, v[j].y); acc.z = f_add(acc.z, v[j].z); acc.w = f_add(acc.w, v[j].w);
      } else {
        acc.x = f_max(acc.x, v[j].x); acc.y = f_max(acc.y, v[j].y); acc.z = f_max(acc.z, v[j].z); acc.w = f_max(acc.w, v[j].w);
      }
    }
    out[i] = acc;
  }
}

}  // namespace

static unsigned grid_for(int64_t n) {
  int64_t b = (n + 255) / 256;
  const int64_t cap = (int64_t)spx_num_sms() * 8;
  if (b > cap) b = cap;
  if (b < 1) b = 1;
  return (unsigned)b;
}

int spx_launch_gather(const spx_gather_params& p, cudaStream_t s, int* nlaunch) {
  if (p.numel <= 0) return 0;
  spx_launch(gather_kernel, dim3(grid_for(p.numel), (unsigned)p.ndev), 256, 0, s, p);
  SPX_CHECK_LAUNCH();
  if (nlaunch) ++*nlaunch;
  return 0;
}

int spx_launch_creduce(const spx_creduce_params& p, cudaStream_t s, int* nlaunch) {
  if (p.numel <= 0) return 0;
  if (p.rank == 1 && p.sstride[0] == 1 && p.numel % 4 == 0 && p.n_members <= 8 && p.ndev == 1) {
    // (the table's pointers are 16-byte aligned: arena buffers are 256 B aligned and chunks are whole float4s)
    spx_launch(creduce_vec_kernel, dim3(grid_for(p.numel / 4), 1u), 256, 0, s, p);
    SPX_CHECK_LAUNCH();
    if (nlaunch) ++*nlaunch;
    return 0;
  }
  spx_launch(creduce_kernel, dim3(grid_for(p.numel), (unsigned)p.ndev), 256, 0, s, p);
  SPX_CHECK_LAUNCH();
  if (nlaunch) ++*nlaunch;
  return 0;
}
