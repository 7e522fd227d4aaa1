// Single-pass batched complex128 FFT for 8192 <= n <= 65536 on a thread-block
// cluster, with TMA (cp.async.bulk.tensor) staging and a persistent,
// double-buffered line loop.
//
//   n = N1 N2, x[n1 N2 + n2] (a line viewed as N1 rows of N2),
//   X[k1 + N1 k2] = sum_n2 W_N2^(n2 k2) W_n^(n2 k1) sum_n1 W_N1^(n1 k1) x[n1 N2 + n2]
//
// A cluster of C CTAs owns one line at a time; CTA r holds the W = N2 / C
// columns [r W, (r+1) W):
//   1. TMA loads the [N1][W] box of the line (rows past in_len are zero
//      filled by the tensor map's bounds) into buffer A[i & 1]; the next
//      line's box is already in flight into the other buffer;
//   2. pass A: W column transforms of length N1 in shared memory (two
//      in-place stages, radix R1a x R2a), optional pointwise factor on load;
//   3. exchange through distributed shared memory: CTA r gathers rows
//      k1 in [r H, (r+1) H), H = N1 / C, of every CTA's columns, applying the
//      twiddle W_n^(n2 k1), into buffer B laid out [N2][H];
//   4. pass B: H row transforms of length N2 in B (radix R1b x R2b);
//   5. one TMA store writes B as the [N2][H] box X[k1 + N1 k2], k1 in the
//      CTA's range.
// HBM sees one read and one write per element (the intermediate never leaves
// the cluster); the copies run on the TMA engine behind the FP64 work.
#include <cooperative_groups.h>
#include <cuda.h>

#include <map>
#include <mutex>
#include <tuple>

#include "fft.cuh"
#include "fft_bfly.cuh"
#include "fft_smem.cuh"

namespace cg = cooperative_groups;

struct ClArgs {
  long long lines;
  long long in_len;  // valid input values per line (zero padded to n)
  int sign;
  const cplx* twN;  // exp(2 pi i k / n)
  const cplx* twA;  // exp(2 pi i k / N1)
  const cplx* twB;  // exp(2 pi i k / N2)
  const cplx* mul = nullptr;  // pointwise factor on load (x * mul_scale * mul[line * mul_ls + e])
  long long mul_ls = 0;
  double mul_scale = 1.0;
};

// phase clock trace of cluster 0 / CTA 0 (diagnostic: tr_debug_cl_trace)
__device__ long long g_cl_trace[8 * 64];
__device__ int g_cl_trace_on = 0;
extern "C" int tr_debug_cl_trace(int enable, long long* out) {
  cudaMemcpyToSymbol(g_cl_trace_on, &enable, sizeof(int));
  if (out) cudaMemcpyFromSymbol(out, g_cl_trace, sizeof(g_cl_trace));
  return 0;
}
#define CL_T(k) \
  if (trace && it < 64) g_cl_trace[it * 8 + (k)] = clock64();

namespace {

TR_D uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

TR_D void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
TR_D void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
TR_D void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
TR_D void tma_load_3d(void* dst, const CUtensorMap* map, int c0, int c1, int c2, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
      "[%5];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}
TR_D void tma_store_3d(const CUtensorMap* map, const void* src, int c0, int c1, int c2) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(map),
               "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2)
               : "memory");
}
TR_D void tma_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
TR_D void tma_wait_read() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
TR_D void tma_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
TR_D void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// stage1 of pass B with the inter-pass twiddle W_n^(n2 k1), k1 = k0 + l:
// for n2 = j2 + R2 j1 it is W_n^(k1 j2) W_n^(k1 R2 j1), the second factor a
// product of at most log2(R1) table powers W_n^(k1 R2 2^b) (independent
// loads, <= 5 roundings) instead of one table load per element.
template <int R1, int R2, int NL, int ES, int NTH>
TR_D void stage1w(cplx* base, int sign, const cplx* twL, const cplx* twN, int k0, unsigned n) {
  constexpr int L = R1 * R2;
  constexpr int NB = R1 <= 1 ? 0 : (R1 <= 2 ? 1 : (R1 <= 4 ? 2 : (R1 <= 8 ? 3 : 4)));
  for (int g = threadIdx.x; g < NL * R2; g += NTH) {
    const int l = g % NL, j2 = g / NL;
    const unsigned k1 = (unsigned)(k0 + l);
    cplx w0 = __ldg(&twN[(k1 * (unsigned)j2) % n]);
    cplx pw[NB > 0 ? NB : 1];
#pragma unroll
    for (int b = 0; b < NB; ++b) pw[b] = __ldg(&twN[(k1 * (unsigned)(R2 << b)) % n]);
    cplx v[R1];
#pragma unroll
    for (int j1 = 0; j1 < R1; ++j1) {
      cplx w = w0;
#pragma unroll
      for (int b = 0; b < NB; ++b)
        if ((j1 >> b) & 1) w = cmul(w, pw[b]);
      if (sign < 0) w.y = -w.y;
      v[j1] = cmul(base[l + (j2 + R2 * j1) * ES], w);
    }
    bfly_any<R1>(v, sign);
    if (j2) {
#pragma unroll
      for (int k1b = 1; k1b < R1; ++k1b) {
        cplx w = __ldg(&twL[(j2 * k1b) % L]);
        if (sign < 0) w.y = -w.y;
        v[k1b] = cmul(v[k1b], w);
      }
    }
#pragma unroll
    for (int k1b = 0; k1b < R1; ++k1b) base[l + (j2 + R2 * k1b) * ES] = v[k1b];
  }
  __syncthreads();
}

TR_D uint32_t mapa(uint32_t addr, int rank) {
  uint32_t out;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(out) : "r"(addr), "r"(rank));
  return out;
}
TR_D void bulk_push(uint32_t dst_cluster, const void* src, uint32_t bytes, uint32_t bar_cluster) {
  asm volatile(
      "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          dst_cluster),
      "r"(smem_u32(src)), "r"(bytes), "r"(bar_cluster)
      : "memory");
}
TR_D void cluster_arrive() { asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory"); }
TR_D void cluster_wait() { asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory"); }

// Buffers (E + N2 complex each): A0 / A1 take the TMA loads ([N1][W] dense)
// and, after pass A, hold C blocks [p][c][k1l] (row pitch H + 1) addressed to
// the CTA p that owns rows k1 in [p H, (p+1) H); B receives the C blocks of
// this CTA (the bulk copies land as [n2][k1l], pitch H + 1) and, after pass
// B, holds the dense [N2][H] output box.
template <int N1, int N2, int C, int R1a, int R2a, int R1b, int R2b, int NTH>
__global__ void __launch_bounds__(NTH, 1)
    fft_cl_kernel(const __grid_constant__ CUtensorMap tin, const __grid_constant__ CUtensorMap tout, ClArgs a) {
  static_assert(N1 == R1a * R2a && N2 == R1b * R2b, "radix split");
  constexpr int W = N2 / C, H = N1 / C, E = N1 * W, HP = H + 1, BLK = W * HP, SZ = E + N2;
  constexpr unsigned n = (unsigned)N1 * N2;
  extern __shared__ __align__(128) unsigned char smraw[];
  cplx* A0 = reinterpret_cast<cplx*>(smraw);
  cplx* A1 = A0 + SZ;
  cplx* B = A1 + SZ;
  uint64_t* bar = reinterpret_cast<uint64_t*>(B + SZ);  // [0], [1]: TMA loads; [2]: incoming blocks
  const int r = (int)cg::this_cluster().block_rank();
  const long long cid = blockIdx.x / C, ncl = gridDim.x / C;
  const int tid = threadIdx.x;
  constexpr uint32_t LOAD_BYTES = (uint32_t)(E * sizeof(cplx));
  constexpr uint32_t BLK_BYTES = (uint32_t)(BLK * sizeof(cplx));

  if (tid == 0) {
    for (int b = 0; b < 3; ++b) mbar_init(&bar[b], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (tid == 0) {
    for (int b = 0; b < 2; ++b) {
      const long long line = cid + b * ncl;
      if (line < a.lines) {
        mbar_expect_tx(&bar[b], LOAD_BYTES);
        tma_load_3d(b ? A1 : A0, &tin, 2 * r * W, 0, (int)line, &bar[b]);
      }
    }
  }
  cluster_arrive();  // barrier phase 0: every CTA's mbarriers are initialised
  cluster_wait();
  const uint32_t b_base = smem_u32(B), bar_b = smem_u32(&bar[2]);
  int it = 0;
  const bool trace = g_cl_trace_on && blockIdx.x == 0 && tid == 0;
  for (long long line = cid; line < a.lines; line += ncl, ++it) {
    const int buf = it & 1;
    cplx* A = buf ? A1 : A0;
    CL_T(0)
    mbar_wait(&bar[buf], (it >> 1) & 1);
    CL_T(1)
    // ---- pass A: W columns of length N1; zero padding past in_len and the
    // pointwise factor on load; outputs to the per-owner blocks
    const cplx* mrow = a.mul ? a.mul + line * a.mul_ls : nullptr;
    const long long in_len = a.in_len;
    const double msc = a.mul_scale;
    stage1<R1a, R2a, W, W, NTH>(A, a.sign, a.twA, [&](int c, int e, cplx x) {
      const long long gi = (long long)e * N2 + r * W + c;
      if (gi >= in_len) return cmk(0.0, 0.0);
      return mrow ? cmul(x, cscale(__ldg(&mrow[gi]), msc)) : x;
    });
    stage2<R1a, R2a, W, W, NTH>(A, a.sign, [&](int c, int k1, cplx v) {
      A[(k1 / H) * BLK + c * HP + (k1 % H)] = v;
    });
    fence_async_smem();  // generic-proxy writes -> the bulk copies read them
    CL_T(2)
    if (it > 0 && tid == 0) tma_wait_read();  // the previous output store has read B
    __syncthreads();
    cluster_arrive();  // all blocks ready, all B buffers free
    cluster_wait();
    CL_T(3)
    if (tid == 0) {
      mbar_expect_tx(&bar[2], C * BLK_BYTES);
      for (int p = 0; p < C; ++p)
        bulk_push(mapa(b_base + r * BLK_BYTES, p), A + p * BLK, BLK_BYTES, mapa(bar_b, p));
    }
    mbar_wait(&bar[2], it & 1);
    CL_T(4)
    cluster_arrive();  // this CTA's incoming blocks are complete
    // ---- pass B: H rows of length N2 (pitch H + 1), twiddle W_n^(n2 k1) on load
    const cplx* twN = a.twN;
    const int sign = a.sign;
    stage1w<R1b, R2b, H, HP, NTH>(B, sign, a.twB, twN, r * H, n);
    stage2<R1b, R2b, H, HP, NTH>(B, sign, [&](int k1l, int k2, cplx v) { B[k2 * H + k1l] = v; });
    CL_T(5)
    cluster_wait();  // every CTA has its blocks: every bulk read of A is done
    if (tid == 0) {
      const long long nxt = line + 2 * ncl;
      if (nxt < a.lines) {
        mbar_expect_tx(&bar[buf], LOAD_BYTES);
        tma_load_3d(A, &tin, 2 * r * W, 0, (int)nxt, &bar[buf]);
      }
    }
    fence_async_smem();
    __syncthreads();
    CL_T(6)
    if (tid == 0) {
      tma_store_3d(&tout, B, 2 * r * H, 0, (int)line);
      tma_commit();
    }
  }
  if (tid == 0) tma_wait_all();
  cluster_arrive();  // no CTA leaves while a partner may still copy into it
  cluster_wait();
}

// ------------------------------------------------------------ host side
typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn encode_fn() {
  static EncodeFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<EncodeFn>(p);
  }();
  return fn;
}

// 3-D map over [lines][rows][row_len] complex values (as doubles), box
// [1][box_rows][box_len]; rows past `rows` read as zero.
int make_map(CUtensorMap* m, const void* base, long long row_len, long long rows, long long row_stride,
             long long lines, long long line_stride, int box_len, int box_rows) {
  EncodeFn enc = encode_fn();
  if (!enc) return -1;
  cuuint64_t dims[3] = {(cuuint64_t)(2 * row_len), (cuuint64_t)rows, (cuuint64_t)lines};
  cuuint64_t strides[2] = {(cuuint64_t)(row_stride * 16), (cuuint64_t)(line_stride * 16)};
  cuuint32_t box[3] = {(cuuint32_t)(2 * box_len), (cuuint32_t)box_rows, 1};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult rc = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<void*>(base), dims, strides, box, es,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return rc == CUDA_SUCCESS ? 0 : -1;
}

struct ClShape {
  int N1, N2, C;
};

template <int N1, int N2, int C, int R1a, int R2a, int R1b, int R2b, int NTH = 256>
int launch_cl(const cplx* in, long long in_ls, long long in_len, cplx* out, long long out_ls, ClArgs a,
              cudaStream_t st) {
  constexpr int W = N2 / C, H = N1 / C;
  CUtensorMap tin, tout;
  // rows past the last (partial) row of in_len read as zero; the partial
  // row's tail is masked in pass A
  a.in_len = in_len;
  if (make_map(&tin, in, N2, (in_len + N2 - 1) / N2, N2, a.lines, in_ls, W, N1)) return -1;
  if (make_map(&tout, out, N1, N2, N1, a.lines, out_ls, H, N2)) return -1;
  auto kern = fft_cl_kernel<N1, N2, C, R1a, R2a, R1b, R2b, NTH>;
  const size_t smem = 3 * sizeof(cplx) * ((size_t)N1 * W + N2) + 64;
  static int max_clusters = -1;
  if (max_clusters < 0) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (C > 8) cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchConfig_t q = {};
    q.gridDim = dim3(C * 64);
    q.blockDim = dim3(NTH);
    q.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = C;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    q.attrs = at;
    q.numAttrs = 1;
    int mc = 0;
    if (cudaOccupancyMaxActiveClusters(&mc, kern, &q) != cudaSuccess || mc < 1) {
      cudaGetLastError();
      mc = 0;
    }
    max_clusters = mc;
  }
  if (max_clusters < 1) return -1;
  const long long ncl = std::min<long long>(max_clusters, a.lines);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(C * ncl));
  cfg.blockDim = dim3(NTH);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = C;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  TrKTimer _kt(TRK_FFT, st);
  if (cudaLaunchKernelEx(&cfg, kern, tin, tout, a) != cudaSuccess) {
    cudaGetLastError();
    return -1;
  }
  return 0;
}

}  // namespace

// Lengths with a cluster kernel (fft_exec routes them here when the input
// stride and zero padding fit the tensor maps).
bool fft_cl_supported(long long n) {
  return n == 8192 || n == 12288 || n == 16384 || n == 32768 || n == 65536;
}

int fft_cl_exec(long long n, const cplx* in, long long in_ls, long long in_len, cplx* out, long long out_ls,
                long long lines, int sign, const cplx* twN, const cplx* mul, long long mul_ls, double mul_scale,
                cudaStream_t st) {
  if (lines <= 0) return 0;
  if (lines > (1LL << 30)) return -1;
  ClArgs a;
  a.lines = lines;
  a.sign = sign;
  a.twN = twN;
  a.mul = mul;
  a.mul_ls = mul_ls;
  a.mul_scale = mul_scale;
  switch (n) {
    case 8192:
      a.twA = twiddle_table(64);
      a.twB = twiddle_table(128);
      return launch_cl<64, 128, 4, 8, 8, 16, 8>(in, in_ls, in_len, out, out_ls, a, st);
    case 12288:
      a.twA = twiddle_table(48);
      a.twB = twiddle_table(256);
      return launch_cl<48, 256, 4, 16, 3, 16, 16>(in, in_ls, in_len, out, out_ls, a, st);
    case 16384:
      a.twA = twiddle_table(128);
      a.twB = twiddle_table(128);
      return launch_cl<128, 128, 4, 16, 8, 16, 8>(in, in_ls, in_len, out, out_ls, a, st);
    case 32768:
      a.twA = twiddle_table(128);
      a.twB = twiddle_table(256);
      return launch_cl<128, 256, 8, 16, 8, 16, 16>(in, in_ls, in_len, out, out_ls, a, st);
    case 65536:
      a.twA = twiddle_table(256);
      a.twB = twiddle_table(256);
      return launch_cl<256, 256, 16, 16, 16, 16, 16>(in, in_ls, in_len, out, out_ls, a, st);
    default:
      return -1;
  }
}
