// Device decode of row-delta coded KJT rows (include/recd_host.h encodes on
// the host).  Per feature: literal count of every row (KEY: L, SHIFT: 1,
// REPEAT: 0) -> exclusive scan -> row r's values are literals
// [c(r) - L_r, c(r)), c the inclusive prefix: a REPEAT row re-reads its
// predecessor's window and a SHIFT row the window one literal further, since
// the new IDs of a run of REPEAT / SHIFT rows follow its KEY row's literals.
//   k_rc_count   literal count per row
//   scan         (recd_prims) exclusive prefix per feature
//   k_rc_copy    value-parallel gather copy literals -> values (k_copy's
//                layout: block per CH values, rows staged in shared memory,
//                fixed-length rows stepped without a search)
#include <algorithm>
#include <vector>

#include "../../include/recd_host.h"
#include "recd_prims.cuh"

namespace recd {
namespace {

constexpr int RC_NT = 256;
constexpr int RC_IT = 16;
constexpr int RC_CH = RC_NT * RC_IT;  // values per block
constexpr int RC_MAXR = 512;          // rows staged per pass

struct RcParams {
  int F;
  int64_t B;
  const uint8_t* codes[RECD_MAX_FEAT];
  const int64_t* offsets[RECD_MAX_FEAT];
  const int64_t* lits[RECD_MAX_FEAT];
  int64_t* out[RECD_MAX_FEAT];
  const int64_t* nv;                   // device [F] value counts
  int64_t blk0[RECD_MAX_FEAT + 1];     // first copy block of each feature
  int64_t* pre;                        // [F][B] literal counts -> exclusive prefix
};

__device__ __forceinline__ int64_t rc_len(const RcParams& p, int f, int64_t r) {
  const int64_t* off = p.offsets[f];
  return ((r + 1 < p.B) ? off[r + 1] : p.nv[f]) - off[r];
}

__device__ __forceinline__ int64_t rc_lits(uint8_t code, int64_t L) {
  return code == RECD_ROW_KEY ? L : (code == RECD_ROW_SHIFT ? 1 : 0);
}

__global__ void k_rc_count(const __grid_constant__ RcParams p) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (int64_t)p.F * p.B) return;
  const int f = (int)(i / p.B);
  const int64_t r = i - (int64_t)f * p.B;
  p.pre[i] = rc_lits(p.codes[f][r], rc_len(p, f, r));
}

__global__ void __launch_bounds__(RC_NT) k_rc_copy(const __grid_constant__ RcParams p) {
  const int f = block_feature(p.blk0, p.F, (int64_t)blockIdx.x);
  const int64_t NV = p.nv[f];
  const int64_t j0 = ((int64_t)blockIdx.x - p.blk0[f]) * RC_CH;
  if (j0 >= NV) return;
  const int64_t j1 = min(NV, j0 + (int64_t)RC_CH);
  const int tid = threadIdx.x;
  const int64_t B = p.B;
  const int64_t* off = p.offsets[f];
  const int64_t* pre = p.pre + (int64_t)f * B;
  const uint8_t* codes = p.codes[f];
  const int64_t* src = p.lits[f];
  int64_t* dst = p.out[f];
  __shared__ int64_t s_r0;
  __shared__ int64_t s_uo[RC_MAXR + 1];  // row starts
  __shared__ int64_t s_so[RC_MAXR];      // row windows in the literals
  if (tid < 32) {
    const int64_t r = warp_last_le(off, B, j0, tid);
    if (tid == 0) s_r0 = r;
  }
  __syncthreads();
  int64_t r0 = s_r0;
  while (true) {
    const int nr = (int)min((int64_t)RC_MAXR, B - r0);
    for (int t = tid; t <= nr; t += RC_NT) {
      const int64_t r = r0 + t;
      const int64_t a = (r < B) ? off[r] : NV;
      s_uo[t] = a;
      if (t < nr) {
        const int64_t L = ((r + 1 < B) ? off[r + 1] : NV) - a;
        s_so[t] = pre[r] + rc_lits(codes[r], L) - L;  // c(r) - L_r
      }
    }
    __syncthreads();
    const int64_t covered = s_uo[nr];
    const int64_t qa = max(j0, s_uo[0]), qb = min(j1, covered);
    const int64_t L0 = nr > 0 ? s_uo[1] - s_uo[0] : 0;
    bool uni = L0 > 0 && L0 < (1 << 23);
    for (int t = tid; t < nr; t += RC_NT) uni &= (s_uo[t + 1] - s_uo[t]) == L0;
    if (__syncthreads_and(uni)) {
      // fixed-length rows: the row of q is stepped, 4 loads in flight
      const uint32_t L = (uint32_t)L0, dj = RC_NT / L, dr = RC_NT % L;
      const int64_t q_first = qa + tid;
      uint32_t r = 0, rem = 0;
      if (q_first < qb) {
        const uint32_t rel = (uint32_t)(q_first - s_uo[0]);
        r = rel / L;
        rem = rel - r * L;
      }
      for (int64_t qq = q_first; qq < qb; qq += 4 * RC_NT) {
        int64_t a[4], v[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          a[k] = s_so[min(r, (uint32_t)(nr - 1))] + rem;
          r += dj;
          rem += dr;
          if (rem >= L) {
            rem -= L;
            ++r;
          }
        }
#pragma unroll
        for (int k = 0; k < 4; ++k)
          if (qq + k * RC_NT < qb) v[k] = __ldg(src + a[k]);
#pragma unroll
        for (int k = 0; k < 4; ++k)
          if (qq + k * RC_NT < qb) dst[qq + k * RC_NT] = v[k];
      }
    } else {
      int r = 0;
      for (int64_t q = qa + tid; q < qb; q += RC_NT) {
        if (s_uo[min(r + 8, nr)] <= q) {
          int lo = r + 8, hi = nr - 1;
          while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (s_uo[mid] <= q) lo = mid; else hi = mid - 1;
          }
          r = lo;
        } else {
          while (s_uo[r + 1] <= q) ++r;
        }
        dst[q] = __ldg(src + s_so[r] + (q - s_uo[r]));
      }
    }
    if (covered >= j1) break;
    __syncthreads();
    r0 += nr;
  }
}

std::vector<ScanDesc> rc_scans(int F, int64_t B, int64_t* pre) {
  std::vector<ScanDesc> d;
  for (int f = 0; f < F; ++f) d.push_back({pre + (int64_t)f * B, pre + (int64_t)f * B, B, nullptr, nullptr});
  return d;
}

size_t rc_carve(void* base, size_t cap, int F, int64_t B, int64_t** pre, int64_t** part) {
  Arena a(base, cap);
  *pre = a.take<int64_t>((size_t)F * B);
  std::vector<ScanDesc> d = rc_scans(F, B, nullptr);
  *part = a.take<int64_t>(std::max<int64_t>(scan_part_words(d.data(), F), 1));
  return a.used;
}

}  // namespace
}  // namespace recd

using namespace recd;

extern "C" size_t recd_rowcode_scratch_bytes(int32_t num_features, int64_t batch_size) {
  if (num_features <= 0 || num_features > RECD_MAX_FEAT || batch_size <= 0) return 0;
  int64_t *pre, *part;
  return rc_carve(nullptr, 0, num_features, batch_size, &pre, &part);
}

extern "C" int recd_rowcode_decode(int32_t num_features, int64_t batch_size,
                                   const uint8_t* const* codes, const int64_t* const* offsets,
                                   const int64_t* num_values, const int64_t* value_caps,
                                   const int64_t* const* lits, int64_t* const* values_out,
                                   void* scratch, size_t scratch_bytes, recd_stream_t stream_) {
  cudaStream_t stream = (cudaStream_t)stream_;
  const int F = num_features;
  const int64_t B = batch_size;
  if (F <= 0 || F > RECD_MAX_FEAT || B <= 0 || !codes || !offsets || !num_values || !value_caps ||
      !lits || !values_out)
    return RECD_ERR_ARG;
  RcParams p;
  memset(&p, 0, sizeof(p));
  p.F = F;
  p.B = B;
  p.nv = num_values;
  int64_t* part = nullptr;
  if (rc_carve(scratch, scratch_bytes, F, B, &p.pre, &part) > scratch_bytes) return RECD_ERR_SCRATCH;
  int64_t blk = 0;
  for (int f = 0; f < F; ++f) {
    if (!codes[f] || !offsets[f] || !lits[f] || !values_out[f]) return RECD_ERR_ARG;
    p.codes[f] = codes[f];
    p.offsets[f] = offsets[f];
    p.lits[f] = lits[f];
    p.out[f] = values_out[f];
    p.blk0[f] = blk;
    blk += std::max<int64_t>(1, ceil_div(value_caps[f], RC_CH));
  }
  p.blk0[F] = blk;
  k_rc_count<<<(unsigned)ceil_div((int64_t)F * B, 256), 256, 0, stream>>>(p);
  std::vector<ScanDesc> d = rc_scans(F, B, p.pre);
  int rc = seg_exclusive_scan(d.data(), F, part, stream);
  if (rc != RECD_OK) return rc;
  k_rc_copy<<<(unsigned)blk, RC_NT, 0, stream>>>(p);
  note_launch(2);
  RECD_LAUNCH_CHECK();
  return RECD_OK;
}
