// Decode-step prologue: rotary position embedding of the new
// tokens' queries and keys, and the append of their K/V into the paged pool,
// in one launch.
//
// Reference: the model computes, per layer and decode step,
//   q = kernels.rope_rows(q, pos, 10000.0); k = kernels.rope_rows(k, pos, ...)
// (model.py:292-293; rope_rows = _kernels_cy.pyx:80-102: consecutive pairs
// (2j, 2j+1) rotated by pos * base^(-2j/d)), then PagedKvCache.append stores
// k and v at the request's next slots (kvcache.py:207-235).  A context
// token's position is its index in the context plus the shared prefix length
// s (context_position, kvcache.py:25-33).
//
// B200 design: a bandwidth-trivial elementwise pass (C2 decode: 1.3 MB), so
// the goal is one launch and exact arithmetic.  One thread owns 8 head dims
// (4 pairs, 16-byte loads / stores).  The angle pos * theta_j and its sine /
// cosine are computed in fp64 like the reference (positions reach 1e5 and
// more: an fp32 angle would be off by up to 1e-2 rad), theta_j = base^(-2j/d)
// from a per-CTA fp64 table; the rotation is done in fp64 and rounded once
// to the output type.
#include "rb_common.cuh"

namespace rb {

constexpr int kRopeThreads = 256;

__device__ __forceinline__ void rope_table(double* theta, int half, int d, double base) {
  for (int j = threadIdx.x; j < half; j += blockDim.x) theta[j] = pow(base, (-2.0 * j) / d);
  __syncthreads();
}

// 8 consecutive elements [e0, e0 + 8) of one row rotated to position pos.
__device__ __forceinline__ void rope8(const float (&x)[8], float (&y)[8], int e0, double pos,
                                      const double* theta) {
#pragma unroll
  for (int p = 0; p < 4; ++p) {
    const double ang = pos * theta[(e0 >> 1) + p];
    double sa, ca;
    sincos(ang, &sa, &ca);
    const double x0 = x[2 * p], x1 = x[2 * p + 1];
    y[2 * p] = static_cast<float>(x0 * ca - x1 * sa);
    y[2 * p + 1] = static_cast<float>(x0 * sa + x1 * ca);
  }
}

__device__ __forceinline__ void load_bf16x8(const __nv_bfloat16* p, float (&x)[8]) {
  const uint4 u = *reinterpret_cast<const uint4*>(p);
  const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const __nv_bfloat162 h = *reinterpret_cast<const __nv_bfloat162*>(&w[i]);
    x[2 * i] = __bfloat162float(h.x);
    x[2 * i + 1] = __bfloat162float(h.y);
  }
}

__device__ __forceinline__ void store_bf16x8(__nv_bfloat16* p, const float (&y)[8]) {
  uint4 u;
  u.x = pack_bf16x2(y[0], y[1]);
  u.y = pack_bf16x2(y[2], y[3]);
  u.z = pack_bf16x2(y[4], y[5]);
  u.w = pack_bf16x2(y[6], y[7]);
  *reinterpret_cast<uint4*>(p) = u;
}

// Work item = (token t, row kind, head, 8-dim chunk c); kinds in order:
// hq query rows (rotated into q_out), hkv key rows (rotated into the pool),
// hkv value rows (copied into the pool).
__global__ void __launch_bounds__(kRopeThreads)
    rope_append_kernel(const __nv_bfloat16* q_in, __nv_bfloat16* q_out,
                       const __nv_bfloat16* __restrict__ k_new,
                       const __nv_bfloat16* __restrict__ v_new,
                       const long long* __restrict__ positions, const int* __restrict__ slots,
                       int n_tok, int hq, int hkv, double base, __nv_bfloat16* k_pool,
                       __nv_bfloat16* v_pool, int block_size, long long stride_block,
                       long long stride_tok, long long stride_head) {
  __shared__ double theta[64];
  rope_table(theta, 64, 128, base);
  const int rows = hq + 2 * hkv;
  const long long total = static_cast<long long>(n_tok) * rows * 16;
  for (long long idx = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; idx < total;
       idx += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int c = static_cast<int>(idx & 15);
    const long long tr = idx >> 4;
    const int r = static_cast<int>(tr % rows);
    const int t = static_cast<int>(tr / rows);
    const double pos = static_cast<double>(__ldg(positions + t));
    float x[8], y[8];
    if (r < hq) {
      const long long off = (static_cast<long long>(t) * hq + r) * 128 + c * 8;
      load_bf16x8(q_in + off, x);
      rope8(x, y, c * 8, pos, theta);
      store_bf16x8(q_out + off, y);
      continue;
    }
    const bool is_v = r >= hq + hkv;
    const int h = is_v ? r - hq - hkv : r - hq;
    const int slot = __ldg(slots + t);
    const long long src = (static_cast<long long>(t) * hkv + h) * 128 + c * 8;
    const long long dst = static_cast<long long>(slot / block_size) * stride_block +
                          static_cast<long long>(slot % block_size) * stride_tok + h * stride_head +
                          c * 8;
    if (is_v) {
      *reinterpret_cast<uint4*>(v_pool + dst) = *reinterpret_cast<const uint4*>(v_new + src);
    } else {
      load_bf16x8(k_new + src, x);
      rope8(x, y, c * 8, pos, theta);
      store_bf16x8(k_pool + dst, y);
    }
  }
}

// fp32 rows of any even width d (<= 1024): the reference's rope_rows.
__global__ void __launch_bounds__(kRopeThreads)
    rope_rows_kernel(const float* x, float* out, const long long* __restrict__ positions,
                     long long n, int d, double base) {
  __shared__ double theta[512];
  const int half = d / 2;
  rope_table(theta, half, d, base);
  const long long total = n * half;
  for (long long idx = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; idx < total;
       idx += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long i = idx / half;
    const int j = static_cast<int>(idx % half);
    const double ang = static_cast<double>(__ldg(positions + i)) * theta[j];
    double sa, ca;
    sincos(ang, &sa, &ca);
    const double x0 = x[i * d + 2 * j], x1 = x[i * d + 2 * j + 1];
    out[i * d + 2 * j] = static_cast<float>(x0 * ca - x1 * sa);
    out[i * d + 2 * j + 1] = static_cast<float>(x0 * sa + x1 * ca);
  }
}

static int rope_grid(long long work) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const long long blocks = (work + kRopeThreads - 1) / kRopeThreads;
  return static_cast<int>(blocks < 4LL * sms ? (blocks > 0 ? blocks : 1) : 4LL * sms);
}

cudaError_t launch_rope_append(const __nv_bfloat16* q_in, __nv_bfloat16* q_out,
                               const __nv_bfloat16* k_new, const __nv_bfloat16* v_new,
                               const long long* positions, const int* slots, int n_tok, int hq,
                               int hkv, double base, __nv_bfloat16* k_pool, __nv_bfloat16* v_pool,
                               int block_size, long long stride_block, long long stride_tok,
                               long long stride_head, cudaStream_t stream) {
  if (n_tok == 0) return cudaSuccess;
  const long long work = static_cast<long long>(n_tok) * (hq + 2 * hkv) * 16;
  rope_append_kernel<<<rope_grid(work), kRopeThreads, 0, stream>>>(
      q_in, q_out, k_new, v_new, positions, slots, n_tok, hq, hkv, base, k_pool, v_pool,
      block_size, stride_block, stride_tok, stride_head);
  return cudaGetLastError();
}

cudaError_t launch_rope_rows(const float* x, float* out, const long long* positions, long long n,
                             int d, double base, cudaStream_t stream) {
  if (n == 0) return cudaSuccess;
  rope_rows_kernel<<<rope_grid(n * (d / 2)), kRopeThreads, 0, stream>>>(x, out, positions, n, d,
                                                                        base);
  return cudaGetLastError();
}

}  // namespace rb
