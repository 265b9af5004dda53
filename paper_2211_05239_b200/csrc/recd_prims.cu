// Segmented stable LSD radix sort + segmented exclusive scan (sm_100a).
//
// Sort: reduce-then-scan per 8-bit digit pass.
//   k_sort_up    block per 16K-element chunk: digit histogram (warp-aggregated
//                shared atomics), stored digit-major per segment [d][chunk].
//   k_sort_scan  block per segment: one exclusive scan over (digit, chunk) in
//                that order gives every chunk's absolute output offset per digit.
//   k_sort_down  block per chunk, 2048-element tiles: per-warp stable ranking
//                with __match_any_sync, tile-local digit bases, staging in shared
//                memory so the scatter writes runs of equal digits contiguously.
// Element order inside a chunk is (tile, warp, round, lane) == input order, so
// every pass is stable and the whole sort is deterministic.
#include <algorithm>
#include <vector>

#include "recd_prims.cuh"

namespace recd {

constexpr int SORT_NT = 256;
#ifndef RECD_SORT_ITEMS
#define RECD_SORT_ITEMS 8
#endif
constexpr int SORT_ITEMS = RECD_SORT_ITEMS;
constexpr int SORT_TILE = SORT_NT * SORT_ITEMS;  // 2048
#ifndef RECD_SORT_CHUNK_TILES
#define RECD_SORT_CHUNK_TILES 8
#endif
#ifndef RECD_SORT_UP_ATOMIC
#define RECD_SORT_UP_ATOMIC 1
#endif
constexpr int SORT_CHUNK = SORT_TILE * RECD_SORT_CHUNK_TILES;  // elements per block
constexpr int SORT_MAXSEG = 64;

struct SortSegDev {
  int64_t base;
  const int64_t* count;
  int64_t chunk0;   // first global chunk of the segment
  int64_t nchunks;  // chunks reserved (capacity-based)
  int64_t hbase;    // first hist word of the segment: 256 * chunk0
};

struct SortParams {
  int S;
  int shift;
  int nbits;
  int64_t total_chunks;
  SortSegDev seg[SORT_MAXSEG];
  const uint32_t* kin;
  const uint32_t* vin;
  uint32_t* kout;
  uint32_t* vout;
  uint32_t* hist;
};

__device__ __forceinline__ int chunk_seg(const SortParams& p, int64_t chunk) {
  int lo = 0, hi = p.S - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (p.seg[mid].chunk0 <= chunk) lo = mid; else hi = mid - 1;
  }
  return lo;
}

__global__ void __launch_bounds__(SORT_NT) k_sort_up(const __grid_constant__ SortParams p) {
  const int64_t chunk = blockIdx.x;
  const int s = chunk_seg(p, chunk);
  const SortSegDev& sg = p.seg[s];
  const int64_t c = chunk - sg.chunk0;
  const int64_t n = *sg.count;
  const int64_t lo = c * SORT_CHUNK;
  if (lo >= n) return;
  const int64_t hi = min(n, lo + (int64_t)SORT_CHUNK);
  const uint32_t mask = (1u << p.nbits) - 1u;
  const uint32_t* k = p.kin + sg.base;
  constexpr int U = 8;  // loads in flight per thread
#if RECD_SORT_UP_ATOMIC
  // per-warp sub-histograms, plain shared atomics (digits of random keys rarely collide)
  __shared__ uint32_t shw[SORT_NT / 32][256];
  const int warp = threadIdx.x >> 5;
#pragma unroll
  for (int w = 0; w < SORT_NT / 32; ++w) shw[w][threadIdx.x] = 0;
  __syncthreads();
  for (int64_t j0 = lo; j0 < hi; j0 += SORT_NT * U) {
    uint32_t kk[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t j = j0 + u * SORT_NT + threadIdx.x;
      kk[u] = j < hi ? __ldg(k + j) : 0u;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t j = j0 + u * SORT_NT + threadIdx.x;
      if (j < hi) atomicAdd(&shw[warp][(kk[u] >> p.shift) & mask], 1u);
    }
  }
  __syncthreads();
  uint32_t tot = 0;
#pragma unroll
  for (int w = 0; w < SORT_NT / 32; ++w) tot += shw[w][threadIdx.x];
  p.hist[sg.hbase + (int64_t)threadIdx.x * sg.nchunks + c] = tot;
#else
  __shared__ uint32_t sh[256];
  sh[threadIdx.x] = 0;
  __syncthreads();
  for (int64_t j0 = lo; j0 < hi; j0 += SORT_NT * U) {
    uint32_t kk[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t j = j0 + u * SORT_NT + threadIdx.x;
      kk[u] = j < hi ? __ldg(k + j) : 0u;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t j = j0 + u * SORT_NT + threadIdx.x;
      const bool valid = j < hi;
      const uint32_t d = valid ? ((kk[u] >> p.shift) & mask) : 0x100u;
      const unsigned peers = __match_any_sync(0xffffffffu, d);
      if (valid && (threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(&sh[d], (uint32_t)__popc(peers));
    }
  }
  __syncthreads();
  p.hist[sg.hbase + (int64_t)threadIdx.x * sg.nchunks + c] = sh[threadIdx.x];
#endif
}

constexpr int SCAN_NT = 1024;
constexpr int SCAN_ITEMS = 8;

// exclusive scan over (digit, chunk) of the active chunks, in place; adds the
// segment base so the downsweep reads absolute output offsets.
__global__ void __launch_bounds__(SCAN_NT) k_sort_scan(const __grid_constant__ SortParams p) {
  const SortSegDev& sg = p.seg[blockIdx.x];
  const int64_t n = *sg.count;
  if (n <= 0) return;
  const int64_t nact = ceil_div(n, SORT_CHUNK);
  const int64_t E = 256 * nact;
  __shared__ int64_t s_scan[32];
  int64_t carry = sg.base;
  for (int64_t tb = 0; tb < E; tb += SCAN_NT * SCAN_ITEMS) {
    const int64_t e0 = tb + (int64_t)threadIdx.x * SCAN_ITEMS;
    uint32_t v[SCAN_ITEMS];
    int64_t sum = 0;
#pragma unroll
    for (int t = 0; t < SCAN_ITEMS; ++t) {
      const int64_t e = e0 + t;
      v[t] = 0;
      if (e < E) {
        const int64_t d = e / nact, c = e - d * nact;
        v[t] = p.hist[sg.hbase + d * sg.nchunks + c];
      }
      sum += v[t];
    }
    int64_t tot;
    int64_t x = carry + block_exclusive_scan<SCAN_NT>(sum, s_scan, &tot);
#pragma unroll
    for (int t = 0; t < SCAN_ITEMS; ++t) {
      const int64_t e = e0 + t;
      if (e < E) {
        const int64_t d = e / nact, c = e - d * nact;
        p.hist[sg.hbase + d * sg.nchunks + c] = (uint32_t)x;
      }
      x += v[t];
    }
    carry += tot;
  }
}

__global__ void __launch_bounds__(SORT_NT) k_sort_down(const __grid_constant__ SortParams p) {
  const int64_t chunk = blockIdx.x;
  const int s = chunk_seg(p, chunk);
  const SortSegDev& sg = p.seg[s];
  const int64_t c = chunk - sg.chunk0;
  const int64_t n = *sg.count;
  const int64_t lo = c * SORT_CHUNK;
  if (lo >= n) return;
  const int64_t hi = min(n, lo + (int64_t)SORT_CHUNK);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t mask = (1u << p.nbits) - 1u;

  __shared__ uint32_t s_off[256];
  __shared__ uint32_t s_wcnt[SORT_NT / 32][256];
  __shared__ uint32_t s_tdb[256];
  __shared__ uint32_t s_keys[SORT_TILE];
  __shared__ uint32_t s_vals[SORT_TILE];
  __shared__ int64_t s_scan[32];

  s_off[tid] = p.hist[sg.hbase + (int64_t)tid * sg.nchunks + c];
  const uint32_t* kin = p.kin + sg.base;
  const uint32_t* vin = p.vin + sg.base;
  const unsigned lt = lanemask_lt();

  for (int64_t tlo = lo; tlo < hi; tlo += SORT_TILE) {
    const int tn = (int)min((int64_t)SORT_TILE, hi - tlo);
    for (int d = lane; d < 256; d += 32) s_wcnt[warp][d] = 0;
    __syncwarp();
    uint32_t key[SORT_ITEMS], val[SORT_ITEMS], rank[SORT_ITEMS];
#pragma unroll
    for (int r = 0; r < SORT_ITEMS; ++r) {  // all loads first: 16 in flight per thread
      const int e = warp * (SORT_TILE / (SORT_NT / 32)) + r * 32 + lane;
      key[r] = e < tn ? __ldg(kin + tlo + e) : 0u;
      val[r] = e < tn ? __ldg(vin + tlo + e) : 0u;
    }
#pragma unroll
    for (int r = 0; r < SORT_ITEMS; ++r) {
      const int e = warp * (SORT_TILE / (SORT_NT / 32)) + r * 32 + lane;
      const bool valid = e < tn;
      const uint32_t d = valid ? ((key[r] >> p.shift) & mask) : 0x100u;
      const unsigned peers = __match_any_sync(0xffffffffu, d);
      uint32_t before = 0;
      if (valid) before = s_wcnt[warp][d];
      __syncwarp();
      if (valid && lane == __ffs(peers) - 1) s_wcnt[warp][d] = before + __popc(peers);
      __syncwarp();
      rank[r] = before + __popc(peers & lt);
    }
    __syncthreads();
    uint32_t tile_cnt = 0;
    {
      const int d = tid;  // SORT_NT == 256 digits
#pragma unroll
      for (int w = 0; w < SORT_NT / 32; ++w) {
        const uint32_t cnt = s_wcnt[w][d];
        s_wcnt[w][d] = tile_cnt;
        tile_cnt += cnt;
      }
    }
    int64_t tot;
    const int64_t tdb = block_exclusive_scan<SORT_NT>(tile_cnt, s_scan, &tot);
    s_tdb[tid] = (uint32_t)tdb;
    __syncthreads();
#pragma unroll
    for (int r = 0; r < SORT_ITEMS; ++r) {
      const int e = warp * (SORT_TILE / (SORT_NT / 32)) + r * 32 + lane;
      if (e < tn) {
        const uint32_t d = (key[r] >> p.shift) & mask;
        const uint32_t lp = s_tdb[d] + s_wcnt[warp][d] + rank[r];
        s_keys[lp] = key[r];
        s_vals[lp] = val[r];
      }
    }
    __syncthreads();
    for (int q = tid; q < tn; q += SORT_NT) {
      const uint32_t k = s_keys[q];
      const uint32_t d = (k >> p.shift) & mask;
      const uint32_t pos = s_off[d] + (uint32_t)q - s_tdb[d];
      p.kout[pos] = k;
      p.vout[pos] = s_vals[q];
    }
    __syncthreads();
    s_off[tid] += tile_cnt;
    __syncthreads();
  }
}

static void build_sort_params(const SegDesc* segs, int S, SortParams* p) {
  memset(p, 0, sizeof(*p));
  p->S = S;
  int64_t chunk = 0;
  for (int s = 0; s < S; ++s) {
    p->seg[s].base = segs[s].base;
    p->seg[s].count = segs[s].count;
    p->seg[s].chunk0 = chunk;
    p->seg[s].nchunks = std::max<int64_t>(1, ceil_div(segs[s].cap, SORT_CHUNK));
    p->seg[s].hbase = 256 * chunk;
    chunk += p->seg[s].nchunks;
  }
  p->total_chunks = chunk;
}

int64_t sort_hist_words(const SegDesc* segs, int S) {
  int64_t words = 0;
  for (int s0 = 0; s0 < S; s0 += SORT_MAXSEG) {
    SortParams p;
    build_sort_params(segs + s0, std::min(SORT_MAXSEG, S - s0), &p);
    words = std::max(words, 256 * p.total_chunks);
  }
  return words;
}

int seg_sort_pairs(const SegDesc* segs, int S, int bits, uint32_t* keys, uint32_t* vals,
                   uint32_t* keys_alt, uint32_t* vals_alt, uint32_t* hist, bool* in_alt,
                   cudaStream_t stream) {
  *in_alt = false;
  if (S <= 0 || bits <= 0) return RECD_OK;
  const int npass = (bits + 7) / 8;
  for (int s0 = 0; s0 < S; s0 += SORT_MAXSEG) {
    SortParams p;
    build_sort_params(segs + s0, std::min(SORT_MAXSEG, S - s0), &p);
    uint32_t *ki = keys, *vi = vals, *ko = keys_alt, *vo = vals_alt;
    for (int pass = 0; pass < npass; ++pass) {
      p.shift = 8 * pass;
      p.nbits = std::min(8, bits - 8 * pass);
      p.kin = ki; p.vin = vi; p.kout = ko; p.vout = vo;
      p.hist = hist;
      k_sort_up<<<(unsigned)p.total_chunks, SORT_NT, 0, stream>>>(p);
      k_sort_scan<<<p.S, SCAN_NT, 0, stream>>>(p);
      k_sort_down<<<(unsigned)p.total_chunks, SORT_NT, 0, stream>>>(p);
      note_launch(3);
      std::swap(ki, ko);
      std::swap(vi, vo);
    }
  }
  *in_alt = (npass % 2) == 1;
  RECD_LAUNCH_CHECK();
  return RECD_OK;
}

// ------------------------------------------------------------------- scan
constexpr int XS_NT = 256;
constexpr int XS_ITEMS = 16;
constexpr int XS_CHUNK = XS_NT * XS_ITEMS;  // 4096
constexpr int XS_MAXSEG = 48;

struct ScanSegDev {
  const int64_t* in;
  int64_t* out;
  int64_t cap;
  const int64_t* count;
  int64_t* total;
  int64_t chunk0;
  int64_t nchunks;
};
struct ScanParams {
  int S;
  int64_t total_chunks;
  ScanSegDev seg[XS_MAXSEG];
  int64_t* part;
};

__device__ __forceinline__ int scan_seg(const ScanParams& p, int64_t chunk) {
  int lo = 0, hi = p.S - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (p.seg[mid].chunk0 <= chunk) lo = mid; else hi = mid - 1;
  }
  return lo;
}

__global__ void __launch_bounds__(XS_NT) k_scan_reduce(const __grid_constant__ ScanParams p) {
  const int64_t chunk = blockIdx.x;
  const ScanSegDev& sg = p.seg[scan_seg(p, chunk)];
  const int64_t n = sg.count ? *sg.count : sg.cap;
  const int64_t lo = (chunk - sg.chunk0) * XS_CHUNK;
  int64_t sum = 0;
  for (int64_t j = lo + threadIdx.x; j < min(n, lo + (int64_t)XS_CHUNK); j += XS_NT) sum += sg.in[j];
  __shared__ int64_t s_scan[32];
  int64_t tot;
  block_exclusive_scan<XS_NT>(sum, s_scan, &tot);
  if (threadIdx.x == 0) p.part[chunk] = tot;
}

__global__ void __launch_bounds__(1024) k_scan_parts(const __grid_constant__ ScanParams p) {
  const ScanSegDev& sg = p.seg[blockIdx.x];
  __shared__ int64_t s_scan[32];
  int64_t carry = 0;
  for (int64_t tb = 0; tb < sg.nchunks; tb += 1024) {
    const int64_t c = tb + threadIdx.x;
    const int64_t v = c < sg.nchunks ? p.part[sg.chunk0 + c] : 0;
    int64_t tot;
    const int64_t x = block_exclusive_scan<1024>(v, s_scan, &tot);
    if (c < sg.nchunks) p.part[sg.chunk0 + c] = carry + x;
    carry += tot;
  }
  if (threadIdx.x == 0 && sg.total) *sg.total = carry;
}

__global__ void __launch_bounds__(XS_NT) k_scan_down(const __grid_constant__ ScanParams p) {
  const int64_t chunk = blockIdx.x;
  const ScanSegDev& sg = p.seg[scan_seg(p, chunk)];
  const int64_t n = sg.count ? *sg.count : sg.cap;
  const int64_t lo = (chunk - sg.chunk0) * XS_CHUNK;
  if (lo >= n) return;
  const int64_t j0 = lo + (int64_t)threadIdx.x * XS_ITEMS;
  int64_t v[XS_ITEMS];
  int64_t sum = 0;
#pragma unroll
  for (int t = 0; t < XS_ITEMS; ++t) {
    v[t] = (j0 + t < n) ? sg.in[j0 + t] : 0;
    sum += v[t];
  }
  __shared__ int64_t s_scan[32];
  int64_t tot;
  int64_t x = p.part[chunk] + block_exclusive_scan<XS_NT>(sum, s_scan, &tot);
#pragma unroll
  for (int t = 0; t < XS_ITEMS; ++t) {
    if (j0 + t < n) sg.out[j0 + t] = x;
    x += v[t];
  }
}

static void build_scan_params(const ScanDesc* segs, int S, ScanParams* p) {
  memset(p, 0, sizeof(*p));
  p->S = S;
  int64_t chunk = 0;
  for (int s = 0; s < S; ++s) {
    p->seg[s].in = segs[s].in;
    p->seg[s].out = segs[s].out;
    p->seg[s].cap = segs[s].cap;
    p->seg[s].count = segs[s].count;
    p->seg[s].total = segs[s].total;
    p->seg[s].chunk0 = chunk;
    p->seg[s].nchunks = std::max<int64_t>(1, ceil_div(segs[s].cap, XS_CHUNK));
    chunk += p->seg[s].nchunks;
  }
  p->total_chunks = chunk;
}

int64_t scan_part_words(const ScanDesc* segs, int S) {
  int64_t words = 0;
  for (int s0 = 0; s0 < S; s0 += XS_MAXSEG) {
    ScanParams p;
    build_scan_params(segs + s0, std::min(XS_MAXSEG, S - s0), &p);
    words = std::max(words, p.total_chunks);
  }
  return words;
}

int seg_exclusive_scan(const ScanDesc* segs, int S, int64_t* part, cudaStream_t stream) {
  for (int s0 = 0; s0 < S; s0 += XS_MAXSEG) {
    ScanParams p;
    build_scan_params(segs + s0, std::min(XS_MAXSEG, S - s0), &p);
    p.part = part;
    k_scan_reduce<<<(unsigned)p.total_chunks, XS_NT, 0, stream>>>(p);
    k_scan_parts<<<p.S, 1024, 0, stream>>>(p);
    k_scan_down<<<(unsigned)p.total_chunks, XS_NT, 0, stream>>>(p);
    note_launch(3);
  }
  RECD_LAUNCH_CHECK();
  return RECD_OK;
}

}  // namespace recd
