// Partial (shift-aware) IKJT of one feature: build_partial_ikjt
// (/root/reference/pkg/src/sessiondedup/tensors.py:311-360) on the GPU,
// bit-exact with the reference's greedy batch-order encoder.
//
// The reference walks the rows in order over one growing value buffer: reuse
// the leftmost aligned occurrence of the row, else append the row minus its
// longest proper prefix that matches the buffer's suffix.  Two facts make it
// parallel:
//  1. A row equal to an earlier row reuses that earlier row's window (the
//     buffer is append-only, and an occurrence left of it would have to
//     straddle the earlier row's buffer end, contradicting the maximal
//     overlap).  So only the U unique rows of recd_dedup (first-occurrence
//     order = the order the greedy meets them) are encoded; batch rows take
//     their unique row's window.
//  2. After a row is appended the buffer ENDS with that whole row.  So, if
//     every unique row is assumed appended, the suffix overlap of row u
//     against the buffer is decided by the previous appended row a alone for
//     k <= |a|: a speculative overlap per row, an exclusive scan of the
//     appended lengths, and one parallel copy build the whole buffer.
// A verification pass then checks each speculated row against the buffer
// prefix it would have seen, E_u elements long: (i) no aligned occurrence in
// buffer[0, E_u) (candidates: the buffer positions in hash(T[0])'s bucket of a
// CSR index built by counting atomics + a scan), (ii) no longer overlap k > |a| reaching past the
// previous row.  The first failing row u* has a correct prefix in front of
// it, so its true decision (found at p / overlap k) is pinned and the next
// round re-speculates the rows after it.  Session-structured batches verify
// in the first round; adversarial ones (rows that are substrings of earlier
// content) cost one round per such row, each round a handful of launches.
//
// Layout: uvalues/uoffsets are recd_dedup's unique rows of the key (offsets
// are row starts), `inverse` its inverse lookup.  Output: the buffer in
// values_out (capacity num_uvalues >= final length), windows_out[B][2],
// *num_values_out (host).  The call synchronises the stream once per round
// (one 16-byte read: buffer length + first failing row); the windows kernel
// is left enqueued.
#include <algorithm>

#include "recd_common.cuh"
#include "recd_prims.cuh"

namespace recd {

enum : int32_t { PK_NONE = 0, PK_FOUND = 1, PK_OV = 2 };

struct PartialParams {
  int64_t U, nval;
  const int64_t* uval;
  const int64_t* uoff;
  int32_t* pin_kind;   // pinned decision of a unique row (PK_*)
  int64_t* pin_val;    // found position / overlap length
  int64_t* ov;         // speculative overlap
  int64_t* app;        // appended length (scan input)
  int64_t* E;          // exclusive scan: buffer length in front of the row
  int64_t* prevn;      // length of the previous appended row (0: none)
  int64_t* ustart;     // window start per unique row
  int64_t* buf;        // the value buffer (values_out)
  // index of the buffer: positions bucketed by hash(value) (CSR)
  int64_t nb;            // buckets (power of two)
  int64_t* bstart;       // counts, then (exclusive scan) bucket starts
  int32_t* bcur;         // fill cursor per bucket
  uint32_t* bidx;        // positions, grouped by bucket
  const int64_t* total;  // device: buffer length
  int32_t* res_kind;
  int64_t* res_val;
  unsigned long long* fail;  // first failing unique row (ctl[1]; ctl[0] = total)
};

__device__ __forceinline__ int64_t pt_len(const PartialParams& p, int64_t u) {
  return (u + 1 < p.U ? p.uoff[u + 1] : p.nval) - p.uoff[u];
}
__device__ __forceinline__ uint32_t pt_hash(int64_t v) { return (uint32_t)(mix64((uint64_t)v) >> 32); }

// x[0, k) == y[0, k), warp-cooperative (all lanes, same arguments)
__device__ __forceinline__ bool warp_equal(const int64_t* x, const int64_t* y, int64_t k, int lane) {
  for (int64_t j0 = 0; j0 < k; j0 += 32) {
    const int64_t j = j0 + lane;
    const bool bad = j < k && x[j] != y[j];
    if (__any_sync(0xffffffffu, bad)) return false;
  }
  return true;
}

// longest k in [klo, khi] with tail[-k:] == T[:k] (tail points one past the
// last element), 0 if none.  First-element filter over 32 k at a time, then a
// cooperative compare of each surviving k, longest first.
__device__ int64_t warp_longest_overlap(const int64_t* tail, const int64_t* T, int64_t klo, int64_t khi,
                                        int lane) {
  const int64_t t0 = T[0];
  for (int64_t k0 = khi; k0 >= klo; k0 -= 32) {
    const int64_t k = k0 - lane;
    unsigned m = __ballot_sync(0xffffffffu, k >= klo && tail[-k] == t0);
    while (m) {
      const int l = __ffs(m) - 1;  // lowest lane = longest k
      m &= m - 1;
      const int64_t kk = k0 - l;
      if (warp_equal(tail - kk, T, kk, lane)) return kk;
    }
  }
  return 0;
}

constexpr int PT_NT = 256, PT_WPB = PT_NT / 32;

__global__ void __launch_bounds__(PT_NT) k_pt_spec(const __grid_constant__ PartialParams p) {
  const int lane = threadIdx.x & 31;
  const int64_t u = (int64_t)blockIdx.x * PT_WPB + (threadIdx.x >> 5);
  if (u >= p.U) return;
  const int64_t n = pt_len(p, u);
  const int kind = p.pin_kind[u];
  int64_t o = 0, an = 0;
  if (n > 0 && kind != PK_FOUND) {
    int64_t a = u - 1;  // previous appended row (empty and found rows append nothing)
    while (a >= 0 && (pt_len(p, a) == 0 || p.pin_kind[a] == PK_FOUND)) --a;
    if (a >= 0) an = pt_len(p, a);
    if (kind == PK_OV) {
      o = p.pin_val[u];
    } else if (a >= 0) {
      const int64_t khi = min(n - 1, an);
      if (khi >= 1) o = warp_longest_overlap(p.uval + p.uoff[a] + an, p.uval + p.uoff[u], 1, khi, lane);
    }
  }
  if (lane == 0) {
    const bool appends = n > 0 && kind != PK_FOUND;
    p.ov[u] = o;
    p.app[u] = appends ? n - o : 0;
    p.prevn[u] = an;
  }
}

// buffer copy of every appended row's tail + the (hash, position) index
__global__ void __launch_bounds__(PT_NT) k_pt_fill(const __grid_constant__ PartialParams p) {
  const int lane = threadIdx.x & 31;
  const int64_t u = (int64_t)blockIdx.x * PT_WPB + (threadIdx.x >> 5);
  if (u >= p.U) return;
  const int64_t n = pt_len(p, u);
  const int kind = p.pin_kind[u];
  if (n == 0 || kind == PK_FOUND) {
    if (lane == 0) p.ustart[u] = n == 0 ? 0 : p.pin_val[u];
    return;
  }
  const int64_t e = p.E[u], o = p.ov[u];
  if (lane == 0) p.ustart[u] = e - o;
  const int64_t* T = p.uval + p.uoff[u];
  for (int64_t j = o + lane; j < n; j += 32) {
    const int64_t q = e + j - o;
    const int64_t v = T[j];
    p.buf[q] = v;
    atomicAdd(reinterpret_cast<unsigned long long*>(p.bstart + (pt_hash(v) & (p.nb - 1))), 1ull);
  }
}

__global__ void __launch_bounds__(PT_NT) k_pt_bucket(const __grid_constant__ PartialParams p) {
  const int64_t q = (int64_t)blockIdx.x * PT_NT + threadIdx.x;
  if (q >= *p.total) return;
  const int64_t b = pt_hash(p.buf[q]) & (p.nb - 1);
  p.bidx[p.bstart[b] + atomicAdd(p.bcur + b, 1)] = (uint32_t)q;
}

__global__ void __launch_bounds__(PT_NT) k_pt_verify(const __grid_constant__ PartialParams p) {
  const int lane = threadIdx.x & 31;
  const int64_t u = (int64_t)blockIdx.x * PT_WPB + (threadIdx.x >> 5);
  if (u >= p.U) return;
  const int64_t n = pt_len(p, u);
  if (n == 0 || p.pin_kind[u] != PK_NONE) return;  // pinned rows are final
  const int64_t e = p.E[u];
  const int64_t* T = p.uval + p.uoff[u];
  int kind = PK_NONE;
  int64_t val = 0;
  if (n <= e) {
    // (i) leftmost aligned occurrence in buf[0, e): every position of T[0]'s
    // bucket is a candidate (unordered: the minimum matching one wins)
    const int64_t b = pt_hash(T[0]) & (p.nb - 1);
    const int64_t lo = p.bstart[b], hi = b + 1 < p.nb ? p.bstart[b + 1] : *p.total;
    const int64_t t0 = T[0];
    int64_t best = INT64_MAX;
    for (int64_t i0 = lo; i0 < hi; i0 += 32) {
      const int64_t i = i0 + lane;
      const int64_t pos = i < hi ? (int64_t)p.bidx[i] : INT64_MAX;
      const bool cand = i < hi && pos + n <= e && p.buf[pos] == t0;
      unsigned m = __ballot_sync(0xffffffffu, cand);
      while (m) {
        const int l = __ffs(m) - 1;
        m &= m - 1;
        const int64_t pp = __shfl_sync(0xffffffffu, pos, l);
        if (pp < best && warp_equal(p.buf + pp, T, n, lane)) best = pp;
      }
    }
    if (best != INT64_MAX) {
      kind = PK_FOUND;
      val = best;
    }
  }
  if (kind == PK_NONE) {
    // (ii) an overlap longer than the previous appended row
    const int64_t pn = p.prevn[u];
    const int64_t khi = min(n - 1, e);
    if (khi > pn) {
      const int64_t k = warp_longest_overlap(p.buf + e, T, pn + 1, khi, lane);
      if (k > 0) {
        kind = PK_OV;
        val = k;
      }
    }
  }
  if (kind != PK_NONE && lane == 0) {
    p.res_kind[u] = kind;
    p.res_val[u] = val;
    atomicMin(p.fail, (unsigned long long)u);
  }
}

__global__ void k_pt_pin(const __grid_constant__ PartialParams p) {
  const unsigned long long f = *p.fail;
  if (f < (unsigned long long)p.U) {
    p.pin_kind[f] = p.res_kind[f];
    p.pin_val[f] = p.res_val[f];
  }
}

__global__ void __launch_bounds__(PT_NT) k_pt_windows(const __grid_constant__ PartialParams p,
                                                      const int64_t* inverse, int64_t B, int64_t* win) {
  const int64_t i = (int64_t)blockIdx.x * PT_NT + threadIdx.x;
  if (i >= B) return;
  const int64_t u = inverse[i];
  const int64_t n = pt_len(p, u);
  win[2 * i] = n == 0 ? 0 : p.ustart[u];
  win[2 * i + 1] = n;
}

struct PtLayout {
  int64_t cap;
  size_t bytes;
};

static size_t pt_carve(PartialParams* p, int64_t U, int64_t nval, void* scratch, size_t cap_bytes,
                       int64_t** part, int64_t** total) {
  Arena a(scratch, cap_bytes);
  const int64_t cap = std::max<int64_t>(nval, 1), uu = std::max<int64_t>(U, 1);
  p->pin_kind = a.take<int32_t>(uu);
  p->res_kind = a.take<int32_t>(uu);
  p->pin_val = a.take<int64_t>(uu);
  p->ov = a.take<int64_t>(uu);
  p->app = a.take<int64_t>(uu);
  p->E = a.take<int64_t>(uu);
  p->prevn = a.take<int64_t>(uu);
  p->ustart = a.take<int64_t>(uu);
  p->res_val = a.take<int64_t>(uu);
  p->nb = std::max<int64_t>((int64_t)next_pow2((uint64_t)cap) / 2, 1);  // ~1 position per bucket
  p->bstart = a.take<int64_t>(p->nb);
  p->bcur = a.take<int32_t>(p->nb);
  p->bidx = a.take<uint32_t>(cap);
  ScanDesc sd{nullptr, nullptr, uu, nullptr, nullptr}, sb{nullptr, nullptr, p->nb, nullptr, nullptr};
  *part = a.take<int64_t>(std::max(scan_part_words(&sd, 1), scan_part_words(&sb, 1)));
  *total = a.take<int64_t>(2);  // [total, fail]: one D2H read per round
  p->fail = reinterpret_cast<unsigned long long*>(*total + 1);
  return a.used;
}

}  // namespace recd

using namespace recd;

extern "C" size_t recd_partial_ikjt_scratch_bytes(int64_t num_unique, int64_t num_uvalues) {
  PartialParams p;
  int64_t *part, *total;
  return pt_carve(&p, num_unique, num_uvalues, nullptr, 0, &part, &total);
}

extern "C" int recd_partial_ikjt(int64_t batch_size, int64_t num_unique, const int64_t* uvalues,
                                 const int64_t* uoffsets, int64_t num_uvalues, const int64_t* inverse,
                                 int64_t* values_out, int64_t* windows_out, int64_t* num_values_out,
                                 int64_t* rounds_out, void* scratch, size_t scratch_bytes,
                                 recd_stream_t stream_) {
  cudaStream_t stream = (cudaStream_t)stream_;
  if (batch_size <= 0 || num_unique <= 0 || num_unique > batch_size || num_uvalues < 0 || !uoffsets ||
      !inverse || !windows_out || !num_values_out || (num_uvalues > 0 && (!uvalues || !values_out)))
    return RECD_ERR_ARG;
  if (num_uvalues > (int64_t)0x3fffffff) return RECD_ERR_UNSUPPORTED;  // 32-bit positions in the index
  if (recd_partial_ikjt_scratch_bytes(num_unique, num_uvalues) > scratch_bytes) return RECD_ERR_SCRATCH;
  PartialParams p;
  int64_t *part, *total;
  pt_carve(&p, num_unique, num_uvalues, scratch, scratch_bytes, &part, &total);
  p.U = num_unique;
  p.nval = num_uvalues;
  p.uval = uvalues;
  p.uoff = uoffsets;
  p.buf = values_out;
  p.total = total;
  RECD_CUDA_CHECK(cudaMemsetAsync(p.pin_kind, 0, sizeof(int32_t) * num_unique, stream));
  const unsigned g = (unsigned)ceil_div(num_unique, PT_WPB);
  ScanDesc sd{p.app, p.E, num_unique, nullptr, total};
  ScanDesc sb{p.bstart, p.bstart, p.nb, nullptr, nullptr};
  int64_t rounds = 0, ctl[2] = {0, -1};
  for (;;) {
    ++rounds;
    k_pt_spec<<<g, PT_NT, 0, stream>>>(p);
    note_launch();
    int rc = seg_exclusive_scan(&sd, 1, part, stream);
    if (rc != RECD_OK) return rc;
    RECD_CUDA_CHECK(cudaMemsetAsync(p.bstart, 0, sizeof(int64_t) * p.nb, stream));
    RECD_CUDA_CHECK(cudaMemsetAsync(p.bcur, 0, sizeof(int32_t) * p.nb, stream));
    k_pt_fill<<<g, PT_NT, 0, stream>>>(p);
    note_launch();
    if (num_uvalues == 0) break;  // every row empty: nothing to verify
    rc = seg_exclusive_scan(&sb, 1, part, stream);
    if (rc != RECD_OK) return rc;
    k_pt_bucket<<<(unsigned)ceil_div(num_uvalues, PT_NT), PT_NT, 0, stream>>>(p);
    note_launch();
    RECD_CUDA_CHECK(cudaMemsetAsync(p.fail, 0xff, sizeof(unsigned long long), stream));
    k_pt_verify<<<g, PT_NT, 0, stream>>>(p);
    k_pt_pin<<<1, 1, 0, stream>>>(p);
    note_launch(2);
    RECD_CUDA_CHECK(cudaMemcpyAsync(ctl, total, sizeof(ctl), cudaMemcpyDeviceToHost, stream));
    RECD_CUDA_CHECK(cudaStreamSynchronize(stream));
    if ((unsigned long long)ctl[1] >= (unsigned long long)num_unique) break;  // all verified
  }
  k_pt_windows<<<(unsigned)ceil_div(batch_size, PT_NT), PT_NT, 0, stream>>>(p, inverse, batch_size,
                                                                            windows_out);
  note_launch();
  RECD_LAUNCH_CHECK();
  *num_values_out = ctl[0];
  if (rounds_out) *rounds_out = rounds;
  return RECD_OK;
}
