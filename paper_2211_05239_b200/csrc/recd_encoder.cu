// Deduplicated sequence encoder (config 4): `attention_pool` of the reference
// (/root/reference/pkg/src/sessiondedup/trainer_sim.py:347-391) evaluated over
// the UNIQUE rows of a grouped IKJT only, then expanded by inverse_lookup.
//
// Per unique row u with tokens x (n x d, the row's lists of every feature of
// the group concatenated, embedding rows of the tables):
//   q, k, v = x W_q, x W_k, x W_v;  P = softmax(q k^T / sqrt(d)) (row-wise,
//   max-subtracted);  out_u = mean_i (P v)_i W_o = (sum_j w_j v_j) W_o with
//   w_j = (1/n) sum_i P_ij;  empty rows give 0.
//
// Kernels:
//   k_enc_gather  warp per unique row: token embeddings -> X (bf16, [N_tok x d]),
//                 token t0(u) = sum_f uoffsets_f[u] (no scan needed)
//   k_gemm_tn     QKV = X [W_q|W_k|W_v] on the tcgen05 tensor cores: persistent
//                 CTAs, W resident in shared memory (128-B swizzle, K-major),
//                 X tiles of 128 tokens double-buffered with cp.async, BF16 x
//                 BF16 -> F32 accumulators in TMEM (M = 128, N = 3d), epilogue
//                 by 8 warps (two per TMEM lane quarter, 64-column halves):
//                 tcgen05.ld -> BF16 -> shared staging -> one 128-byte bulk
//                 (TMA-engine) store per thread and chunk
//   k_enc_attn    CTA per unique row: scores on the tensor cores (mma.sync
//                 m16n8k16, 64 x 64 blocks), pass 1 row max / sum, pass 2
//                 column sums of P, then (w v) / n and @ W_o in fp32
// Only the QKV projection is GEMM-shaped at scale (N_tok x d x 3d); the per-row
// attention is small (n x n x d per unique row).
#include <algorithm>
#include <cuda_bf16.h>

#include "recd_common.cuh"
#include "recd_umma.cuh"

namespace recd {

// ----------------------------------------------------------------- gather
struct EncParams {
  int F, D;
  int64_t B;
  const float* tables[RECD_MAX_FEAT];
  int64_t table_rows[RECD_MAX_FEAT];
  const int64_t* uvalues[RECD_MAX_FEAT];
  const int64_t* uoffsets[RECD_MAX_FEAT];
  const int64_t* counts;  // device [2F]
  __nv_bfloat16* X;       // [tok cap][D]
  const __nv_bfloat16* QKV;  // [tok cap][3D]
  const float* w_o;       // [D][D]
  float* out;             // [B][D]
  int64_t* err;
};

__device__ __forceinline__ void row_span(const EncParams& p, int f, int64_t u, int64_t U,
                                         int64_t* a, int64_t* e) {
  const int64_t* uo = p.uoffsets[f];
  *a = uo[u];
  *e = (u + 1 < U) ? uo[u + 1] : p.counts[p.F + f];
}

__global__ void __launch_bounds__(256) k_enc_gather(const __grid_constant__ EncParams p) {
  const int lane = threadIdx.x & 31;
  const int64_t U = p.counts[0];
  const int64_t nw = (int64_t)gridDim.x * 8;
  for (int64_t u = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5); u < U; u += nw) {
    int64_t t = 0;
    for (int f = 0; f < p.F; ++f) t += p.uoffsets[f][u];
    for (int f = 0; f < p.F; ++f) {
      int64_t a, e;
      row_span(p, f, u, U, &a, &e);
      const float* W = p.tables[f];
      for (int64_t j = a; j < e; ++j, ++t) {
        const int64_t id = __ldg(p.uvalues[f] + j);
        __nv_bfloat16* dst = p.X + t * p.D;
        if ((uint64_t)id >= (uint64_t)p.table_rows[f]) {
          if (lane == 0) atomicMin(reinterpret_cast<unsigned long long*>(p.err),
                                   (unsigned long long)(((int64_t)f << 40) + j));
          for (int c = lane * 4; c < p.D; c += 128)
            *reinterpret_cast<uint2*>(dst + c) = make_uint2(0u, 0u);
          continue;
        }
        const float* src = W + (uint64_t)id * p.D;
        for (int c = lane * 4; c < p.D; c += 128) {
          const float4 x = __ldg(reinterpret_cast<const float4*>(src + c));
          __nv_bfloat162 lo = __floats2bfloat162_rn(x.x, x.y), hi = __floats2bfloat162_rn(x.z, x.w);
          *reinterpret_cast<uint2*>(dst + c) =
              make_uint2(*reinterpret_cast<uint32_t*>(&lo), *reinterpret_cast<uint32_t*>(&hi));
        }
      }
    }
  }
}

// ------------------------------------------------------- tcgen05 GEMM (TN)
// C[m][n] = sum_k A[m][k] B[n][k], A [M x K], B [N x K], C [M x N], all bf16
// row-major; M (device count) arbitrary, K in {64, 128}, N % 16 == 0, N <= 512.
struct GemmParams {
  const __nv_bfloat16* A;
  const __nv_bfloat16* B;
  __nv_bfloat16* C;
  const int64_t* m_counts;  // M = sum of m_counts[0 .. m_nc)
  int m_nc;
};

__device__ __forceinline__ void cp16_zfill(uint32_t saddr, const void* g, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(saddr), "l"(g),
               "r"(valid ? 16 : 0));
}

constexpr int GM_NT = 256;
constexpr int GM_CPITCH = 272;  // staging row pitch (256 B + 16: conflict-free 16-B stores)  // 8 warps: warps w and w + 4 share TMEM lanes 32 (w % 4) .. + 32
template <int N, int K>
__global__ void __launch_bounds__(GM_NT, 1) k_gemm_tn(const __grid_constant__ GemmParams p) {
  static_assert(K % 64 == 0 && N % 16 == 0 && N <= 512, "tile shape");
  constexpr int KB = K / 64;               // 128-byte K blocks
  constexpr uint32_t A_STAGE = KB * 128 * 128;
  constexpr uint32_t B_BYTES = KB * N * 128;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-B alignment of the swizzle atoms (dynamic smem base is only 16-B aligned)
  uint8_t* smem = smem_raw + ((1024u - ((uint32_t)__cvta_generic_to_shared(smem_raw) & 1023u)) & 1023u);
  uint8_t* sB = smem;
  uint8_t* sA = smem + B_BYTES;
  uint8_t* sC = sA + 2 * A_STAGE;  // epilogue staging: 128 rows x 256 B, padded pitch
  __shared__ __align__(8) uint64_t mbar2[2];
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  int64_t M = 0;
  for (int i = 0; i < p.m_nc; ++i) M += p.m_counts[i];
  const int64_t ntiles = (M + 127) / 128;
  if ((int64_t)blockIdx.x >= ntiles) return;

  if (warp == 0) umma::tmem_alloc<512>(&tmem_base);
  if (tid == 0) {
    umma::mbar_init(&mbar2[0], 1);
    umma::mbar_init(&mbar2[1], 1);
  }
  const uint32_t sB_addr = (uint32_t)__cvta_generic_to_shared(sB);
  const uint32_t sA_addr = (uint32_t)__cvta_generic_to_shared(sA);
  // B once: (row n, K block kb, 16-B chunk c)
  for (int idx = tid; idx < N * KB * 8; idx += GM_NT) {
    const int n = idx / (KB * 8), r = idx - n * (KB * 8), kb = r >> 3, c = r & 7;
    cp16_zfill(sB_addr + kb * N * 128 + umma::sw128_offset(n, c), p.B + (int64_t)n * K + kb * 64 + c * 8,
               true);
  }
  auto load_a = [&](int64_t t, int stage) {
    for (int idx = tid; idx < 128 * KB * 8; idx += GM_NT) {
      const int r = idx / (KB * 8), q = idx - r * (KB * 8), kb = q >> 3, c = q & 7;
      const int64_t m = t * 128 + r;
      const bool ok = m < M;
      cp16_zfill(sA_addr + stage * A_STAGE + kb * 16384 + umma::sw128_offset(r, c),
                 p.A + (ok ? m : 0) * K + kb * 64 + c * 8, ok);
    }
    cp_async_commit();
  };
  load_a(blockIdx.x, 0);
  umma::fence_before_sync();
  __syncthreads();
  umma::fence_after_sync();
  const uint32_t tmem = tmem_base;
  uint32_t phase = 0;
  int stage = 0;
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, stage ^= 1) {
    if (t + gridDim.x < ntiles) load_a(t + gridDim.x, stage ^ 1);
    else cp_async_commit();
    cp_async_wait<1>();  // B and this tile's A (this thread's copies)
    umma::fence_proxy_async();
    __syncthreads();
    // two MMA groups, each committed to its own mbarrier: columns [0, 128)
    // first, so the epilogue of that chunk overlaps the MMAs of the rest
    constexpr int NH = N < 128 ? N : 128;
    if (tid == 0) {
      umma::fence_after_sync();
#pragma unroll
      for (int grp = 0; grp < 2; ++grp) {
        const int cbeg = grp == 0 ? 0 : NH, cend = grp == 0 ? NH : N;
#pragma unroll
        for (int kb = 0; kb < KB; ++kb)
#pragma unroll
          for (int k = 0; k < 4; ++k) {  // UMMA_K = 16 bf16 = 32 B along the swizzled row
            const uint64_t ad = umma::smem_desc_sw128_kmajor(sA_addr + stage * A_STAGE + kb * 16384 + k * 32);
            for (int n0 = cbeg; n0 < cend; n0 += 256) {
              const int nc = (cend - n0) < 256 ? (cend - n0) : 256;
              const uint64_t bd = umma::smem_desc_sw128_kmajor(sB_addr + kb * N * 128 + n0 * 128 + k * 32);
              umma::mma_bf16(tmem + n0, ad, bd, umma::idesc_bf16_f32(128, nc), (kb | k) != 0);
            }
          }
        if (grp == 0 || NH < N) umma::commit(&mbar2[grp]);
      }
    }
    umma::mbar_wait(&mbar2[0], phase);
    umma::fence_after_sync();
    const int lq = warp & 3;  // TMEM lane quarter of this warp
    const int r = lq * 32 + lane;  // tile row of this thread
    const int64_t m = t * 128 + r;
    const int h = warp >> 2;  // the two warps of a lane quarter take the two 64-column halves
    uint8_t* srow = sC + r * GM_CPITCH + h * 128;
#pragma unroll 1
    for (int c0 = 0; c0 < N; c0 += 128) {
      if (c0 == NH && NH < N) {  // the remaining columns' MMAs
        umma::mbar_wait(&mbar2[1], phase);
        umma::fence_after_sync();
      }
      const int cb = c0 + h * 64;  // 64 columns of this thread
      if (cb < N) {
        // staging row segment free again (this thread's previous bulk store read it)
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          float v[32];
          umma::tmem_ld32(tmem + ((uint32_t)(lq * 32) << 16) + cb + 32 * q, v);
          uint32_t w[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            __nv_bfloat162 hh = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);
            w[i] = *reinterpret_cast<uint32_t*>(&hh);
          }
          uint4* dst = reinterpret_cast<uint4*>(srow + q * 64);
#pragma unroll
          for (int i = 0; i < 4; ++i) dst[i] = make_uint4(w[4 * i], w[4 * i + 1], w[4 * i + 2], w[4 * i + 3]);
        }
        // 128 contiguous bytes of row m: one bulk (TMA-engine) store per thread
        umma::fence_proxy_async();
        if (m < M) {
          asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], 128;" ::"l"(p.C + m * N + cb),
                       "r"((uint32_t)__cvta_generic_to_shared(srow))
                       : "memory");
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
      }
    }
    phase ^= 1;
    umma::fence_before_sync();
    __syncthreads();  // TMEM drained and the A stage free before the next tile's MMAs / loads
  }
  cp_async_wait<0>();
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  if (warp == 0) {
    umma::fence_after_sync();
    umma::tmem_free<512>(tmem);
  }
}

// ------------------------------------------------------ per-row attention
constexpr int AT_NT = 128;  // 4 warps, 16 query rows each
constexpr int AT_QB = 64;   // query rows per block
constexpr int AT_KB = 64;   // keys per block

__device__ __forceinline__ void mma16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0,
                                         uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, "
      "{%8, %9}, {%0, %1, %2, %3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// S (16 rows of this warp x 64 keys) = Q_blk K_blk^T, rows / keys from shared
// memory with a row pitch of `pitch` bf16
template <int D>
__device__ __forceinline__ void scores16x64(const __nv_bfloat16* sQ, const __nv_bfloat16* sK, int pitch,
                                            int warp, int lane, float (&s)[8][4]) {
  const int g = lane >> 2, tq = lane & 3;
#pragma unroll
  for (int nt = 0; nt < 8; ++nt)
#pragma unroll
    for (int i = 0; i < 4; ++i) s[nt][i] = 0.f;
  const __nv_bfloat16* q0 = sQ + (warp * 16 + g) * pitch;
  const __nv_bfloat16* q1 = q0 + 8 * pitch;
#pragma unroll
  for (int k0 = 0; k0 < D; k0 += 16) {
    uint32_t a[4];
    a[0] = *reinterpret_cast<const uint32_t*>(q0 + k0 + 2 * tq);
    a[1] = *reinterpret_cast<const uint32_t*>(q1 + k0 + 2 * tq);
    a[2] = *reinterpret_cast<const uint32_t*>(q0 + k0 + 8 + 2 * tq);
    a[3] = *reinterpret_cast<const uint32_t*>(q1 + k0 + 8 + 2 * tq);
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) {
      const __nv_bfloat16* kr = sK + (nt * 8 + g) * pitch + k0;
      mma16816(s[nt], a, *reinterpret_cast<const uint32_t*>(kr + 2 * tq),
               *reinterpret_cast<const uint32_t*>(kr + 8 + 2 * tq));
    }
  }
}

template <int D>
__global__ void __launch_bounds__(AT_NT) k_enc_attn(const __grid_constant__ EncParams p) {
  constexpr int PITCH = D + 8;  // bf16; +16 B per row against bank conflicts
  __shared__ __align__(16) __nv_bfloat16 sQ[AT_QB * PITCH];
  __shared__ __align__(16) __nv_bfloat16 sK[AT_KB * PITCH];
  __shared__ float s_w[1024];  // column sums of P for keys of the current pass (n <= 1024 per chunk)
  __shared__ float s_ctx[D];
  __shared__ float s_wp[AT_NT / 32][AT_KB];  // per-warp column sums of one key block
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, tq = lane & 3;
  const int64_t U = p.counts[0];
  const float scale = 1.0f / sqrtf((float)D);
  for (int64_t u = blockIdx.x; u < U; u += gridDim.x) {
    int64_t t0 = 0, n = 0;
    for (int f = 0; f < p.F; ++f) {
      int64_t a, e;
      row_span(p, f, u, U, &a, &e);
      t0 += a;
      n += e - a;
    }
    float* orow = p.out + u * D;
    if (n == 0) {
      for (int c = tid; c < D; c += AT_NT) orow[c] = 0.f;
      continue;
    }
    const __nv_bfloat16* Q = p.QKV + t0 * (3 * D);
    const __nv_bfloat16* Kg = Q + D;
    const __nv_bfloat16* Vg = Q + 2 * D;
    for (int c = tid; c < D; c += AT_NT) s_ctx[c] = 0.f;
    // key chunks of <= 1024 keys: column sums of P for the chunk, folded into ctx
    for (int64_t kc0 = 0; kc0 < n; kc0 += 1024) {
      const int kcn = (int)min((int64_t)1024, n - kc0);
      for (int j = tid; j < kcn; j += AT_NT) s_w[j] = 0.f;
      for (int64_t q0 = 0; q0 < n; q0 += AT_QB) {
        __syncthreads();
        for (int idx = tid; idx < AT_QB * (D / 8); idx += AT_NT) {  // Q block (16-B chunks)
          const int r = idx / (D / 8), c = idx - r * (D / 8);
          uint4 v = make_uint4(0, 0, 0, 0);
          if (q0 + r < n) v = *reinterpret_cast<const uint4*>(Q + (q0 + r) * (3 * D) + c * 8);
          *reinterpret_cast<uint4*>(sQ + r * PITCH + c * 8) = v;
        }
        // pass 1 over ALL keys: running row max / sum (exact softmax statistics)
        float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;  // rows g, g + 8 of this warp
        // one 64 x 64 block (n <= 64, the common history length): pass 2 reuses
        // pass 1's scaled scores instead of reloading K and recomputing them
        const bool single = n <= AT_KB;
        float s[8][4];
        for (int pass = 0; pass < 2; ++pass) {
          const int64_t kbeg = pass == 0 ? 0 : kc0, kend = pass == 0 ? n : kc0 + kcn;
          for (int64_t k0 = kbeg; k0 < kend; k0 += AT_KB) {
            if (!(single && pass == 1)) {
              __syncthreads();
              for (int idx = tid; idx < AT_KB * (D / 8); idx += AT_NT) {
                const int r = idx / (D / 8), c = idx - r * (D / 8);
                uint4 v = make_uint4(0, 0, 0, 0);
                if (k0 + r < kend) v = *reinterpret_cast<const uint4*>(Kg + (k0 + r) * (3 * D) + c * 8);
                *reinterpret_cast<uint4*>(sK + r * PITCH + c * 8) = v;
              }
              __syncthreads();
              scores16x64<D>(sQ, sK, PITCH, warp, lane, s);
            }
            // C fragment: s[nt][0..1] row g cols nt*8 + 2tq + {0,1}; s[nt][2..3] row g + 8
            if (pass == 0) {
              float bm0 = -INFINITY, bm1 = -INFINITY;
#pragma unroll
              for (int nt = 0; nt < 8; ++nt)
#pragma unroll
                for (int i = 0; i < 2; ++i) {
                  const bool ok = k0 + nt * 8 + 2 * tq + i < kend;
                  s[nt][i] = ok ? s[nt][i] * scale : -INFINITY;
                  s[nt][2 + i] = ok ? s[nt][2 + i] * scale : -INFINITY;
                  bm0 = fmaxf(bm0, s[nt][i]);
                  bm1 = fmaxf(bm1, s[nt][2 + i]);
                }
#pragma unroll
              for (int d = 1; d < 4; d <<= 1) {
                bm0 = fmaxf(bm0, __shfl_xor_sync(0xffffffffu, bm0, d));
                bm1 = fmaxf(bm1, __shfl_xor_sync(0xffffffffu, bm1, d));
              }
              const float nm0 = fmaxf(m0, bm0), nm1 = fmaxf(m1, bm1);
              float a0 = 0.f, a1 = 0.f;
#pragma unroll
              for (int nt = 0; nt < 8; ++nt)
#pragma unroll
                for (int i = 0; i < 2; ++i) {
                  a0 += __expf(s[nt][i] - nm0);
                  a1 += __expf(s[nt][2 + i] - nm1);
                }
#pragma unroll
              for (int d = 1; d < 4; d <<= 1) {
                a0 += __shfl_xor_sync(0xffffffffu, a0, d);
                a1 += __shfl_xor_sync(0xffffffffu, a1, d);
              }
              l0 = l0 * __expf(m0 - nm0) + a0;
              l1 = l1 * __expf(m1 - nm1) + a1;
              m0 = nm0;
              m1 = nm1;
            } else {
              // P_ij = exp(s_ij - m_i) / l_i over valid rows; column sums
              const bool r0 = q0 + warp * 16 + g < n, r1 = q0 + warp * 16 + g + 8 < n;
              const float i0 = r0 ? 1.f / l0 : 0.f, i1 = r1 ? 1.f / l1 : 0.f;
#pragma unroll
              for (int nt = 0; nt < 8; ++nt)
#pragma unroll
                for (int i = 0; i < 2; ++i) {
                  const int64_t j = k0 + nt * 8 + 2 * tq + i;
                  float c = 0.f;
                  if (j < kend) {  // single: s already scaled (same fp32 value)
                    const float s0 = single ? s[nt][i] : s[nt][i] * scale;
                    const float s1 = single ? s[nt][2 + i] : s[nt][2 + i] * scale;
                    c = (r0 ? __expf(s0 - m0) * i0 : 0.f) + (r1 ? __expf(s1 - m1) * i1 : 0.f);
                  }
                  // sum over the 8 row groups (lanes with equal tq)
#pragma unroll
                  for (int d = 4; d < 32; d <<= 1) c += __shfl_xor_sync(0xffffffffu, c, d);
                  if (g == 0) s_wp[warp][nt * 8 + 2 * tq + i] = c;
                }
              __syncthreads();
              // fixed-order sum over the 4 warps' query rows: deterministic, so
              // a unique row encodes identically wherever it occurs
              if (tid < AT_KB && k0 + tid < kend)
                s_w[k0 + tid - kc0] += ((s_wp[0][tid] + s_wp[1][tid]) + s_wp[2][tid]) + s_wp[3][tid];
            }
          }
        }
      }
      __syncthreads();
      // ctx += sum_j w_j v_j over the chunk's keys
      for (int c = tid; c < D; c += AT_NT) {
        float acc = 0.f;
        for (int j = 0; j < kcn; ++j) acc += s_w[j] * __bfloat162float(Vg[(kc0 + j) * (3 * D) + c]);
        s_ctx[c] += acc;
      }
      __syncthreads();
    }
    // out = (ctx / n) W_o
    const float inv_n = 1.f / (float)n;
    for (int c = tid; c < D; c += AT_NT) {
      float acc = 0.f;
      for (int k = 0; k < D; ++k) acc += s_ctx[k] * __ldg(p.w_o + k * D + c);
      orow[c] = acc * inv_n;
    }
    __syncthreads();
  }
}

struct EncScratch {
  __nv_bfloat16* X;
  __nv_bfloat16* QKV;
};
static size_t carve_enc(void* base, size_t cap, int64_t tok_cap, int D, EncScratch* s) {
  Arena a(base, cap);
  s->X = a.take<__nv_bfloat16>((size_t)std::max<int64_t>(tok_cap, 1) * D);
  s->QKV = a.take<__nv_bfloat16>((size_t)std::max<int64_t>(tok_cap, 1) * 3 * D);
  return a.used;
}

template <int N, int K>
static int launch_gemm(const GemmParams& g, cudaStream_t stream) {
  constexpr int smem = (K / 64) * N * 128 + 2 * (K / 64) * 128 * 128 + 128 * GM_CPITCH + 1024;
  RECD_CUDA_CHECK(cudaFuncSetAttribute(k_gemm_tn<N, K>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  k_gemm_tn<N, K><<<num_sms(), GM_NT, smem, stream>>>(g);
  return RECD_OK;
}

}  // namespace recd

using namespace recd;

extern "C" size_t recd_attention_pool_scratch_bytes(int32_t num_features, int32_t dim,
                                                   const int64_t* value_caps) {
  if (num_features <= 0 || num_features > RECD_MAX_FEAT || !value_caps) return 0;
  int64_t tok = 0;
  for (int f = 0; f < num_features; ++f) tok += value_caps[f];
  EncScratch s;
  return carve_enc(nullptr, 0, tok, dim, &s);
}

extern "C" int recd_attention_pool(int32_t num_features, int64_t batch_size, int32_t dim,
                                   const float* const* tables, const int64_t* table_rows,
                                   const int64_t* const* uvalues, const int64_t* const* uoffsets,
                                   const int64_t* value_caps, const int64_t* counts,
                                   const void* w_qkv_t, const float* w_o, float* out, int64_t* err,
                                   void* scratch, size_t scratch_bytes, recd_stream_t stream_) {
  cudaStream_t stream = (cudaStream_t)stream_;
  if (num_features <= 0 || num_features > RECD_MAX_FEAT || batch_size <= 0 || !counts || !w_qkv_t ||
      !w_o || !out || !err || !value_caps)
    return RECD_ERR_ARG;
  if (dim != 64 && dim != 128) return RECD_ERR_UNSUPPORTED;
  EncParams p;
  memset(&p, 0, sizeof(p));
  p.F = num_features;
  p.D = dim;
  p.B = batch_size;
  p.counts = counts;
  int64_t tok = 0;
  for (int f = 0; f < num_features; ++f) {
    if (!tables[f] || !uvalues[f] || !uoffsets[f] || table_rows[f] <= 0) return RECD_ERR_ARG;
    if ((uintptr_t)tables[f] % 16) return RECD_ERR_ARG;
    p.tables[f] = tables[f];
    p.table_rows[f] = table_rows[f];
    p.uvalues[f] = uvalues[f];
    p.uoffsets[f] = uoffsets[f];
    tok += value_caps[f];
  }
  EncScratch s;
  if (carve_enc(scratch, scratch_bytes, tok, dim, &s) > scratch_bytes) return RECD_ERR_SCRATCH;
  p.X = s.X;
  p.QKV = s.QKV;
  p.w_o = w_o;
  p.out = out;
  p.err = err;
  RECD_CUDA_CHECK(cudaMemsetAsync(err, 0x7f, sizeof(int64_t), stream));
  k_enc_gather<<<num_sms() * 8, 256, 0, stream>>>(p);
  GemmParams g;
  g.A = s.X;
  g.B = reinterpret_cast<const __nv_bfloat16*>(w_qkv_t);
  g.C = s.QKV;
  g.m_counts = counts + num_features;  // tokens = sum_f N_u(f)
  g.m_nc = num_features;
  int rc = dim == 64 ? launch_gemm<192, 64>(g, stream) : launch_gemm<384, 128>(g, stream);
  if (rc != RECD_OK) return rc;
  if (dim == 64)
    k_enc_attn<64><<<num_sms() * 8, AT_NT, 0, stream>>>(p);
  else
    k_enc_attn<128><<<num_sms() * 8, AT_NT, 0, stream>>>(p);
  note_launch(3);
  RECD_LAUNCH_CHECK();
  return RECD_OK;
}

// Plain GEMM entry (tests / reuse): C = A B^T, bf16, M rows given on the device.
extern "C" int recd_gemm_bf16_tn(int32_t n, int32_t k, const void* a, const void* b, void* c,
                                 const int64_t* m_count, recd_stream_t stream_) {
  GemmParams g;
  g.A = reinterpret_cast<const __nv_bfloat16*>(a);
  g.B = reinterpret_cast<const __nv_bfloat16*>(b);
  g.C = reinterpret_cast<__nv_bfloat16*>(c);
  g.m_counts = m_count;
  g.m_nc = 1;
  cudaStream_t stream = (cudaStream_t)stream_;
  int rc;
  if (n == 192 && k == 64) rc = launch_gemm<192, 64>(g, stream);
  else if (n == 384 && k == 128) rc = launch_gemm<384, 128>(g, stream);
  else if (n == 128 && k == 128) rc = launch_gemm<128, 128>(g, stream);
  else return RECD_ERR_UNSUPPORTED;
  note_launch();
  if (rc != RECD_OK) return rc;
  RECD_LAUNCH_CHECK();
  return RECD_OK;
}
