// esc_sort.cuh — the framework's own device sort and grouping, included by esc_kernels.cu (no
// library kernels on these paths):
//
//   esc_sort_pairs   stable LSD radix sort of 32- or 64-bit unsigned keys (+ optional 64-bit
//                    values): one histogram launch for every digit pass, then ONE launch per pass
//                    ("onesweep": tile ranks by warp match, a windowed decoupled look-back per
//                    digit across tiles, a shared-memory staged scatter so the writes are runs)
//   esc_runs         the runs of a sorted key array: run starts / sizes / keys (decoded to int64),
//                    the run of every element, and the statistics {runs, first key, last key,
//                    largest run} — one launch (tile flags + a windowed look-back) + a finish
//
// Uses: the hash build's grouping (f1, reference np.unique + stable argsort,
// executor.py:275-303), the CSV loader's TEXT dictionary by first appearance (f3, reference
// storage.py:247-275 / Dictionary.encode), the histogram arm's value sort (f4, reference
// catalog.py:178-223 np.sort).  Stability is the contract that matters: equal keys keep input
// order, so a group's rows stay ascending exactly like numpy's stable argsort.
#pragma once

namespace esc {

constexpr int kSortThreads = 256;
constexpr int kSortItems = 8;
constexpr int kSortTile = kSortThreads * kSortItems;  // elements per tile
constexpr int kSortMaxPasses = 8;
constexpr int kSortWindow = 8;  // look-back: predecessor words in flight per digit thread
// status word of (tile, digit): [tag 16][flag 2][value 46]; tag = this call's pass id
constexpr unsigned long long kSortAgg = 1ull, kSortPre = 2ull;
constexpr unsigned long long kSortValMask = (1ull << 46) - 1;

struct SortPass {
  const void* keys_in;
  const unsigned long long* vals_in;  // nullptr: keys only
  void* keys_out;
  unsigned long long* vals_out;
  int64_t n;
  int32_t shift;
  int32_t pad;
  const uint32_t* hist;          // this pass's 256 global digit counts
  unsigned long long* status;    // [tiles][256]
  unsigned long long* ticket;    // this pass's tile ticket (zero at launch)
  unsigned long long tag;        // pass tag << 48
};

// every pass's digit histogram in one read of the keys (per-block shared counters, then global)
template <typename K>
__global__ void __launch_bounds__(256) sort_hist_kernel(const K* __restrict__ keys, int64_t n, int begin_bit,
                                                        int passes, uint32_t* __restrict__ hist) {
  __shared__ uint32_t h[kSortMaxPasses * 256];
  for (int i = threadIdx.x; i < passes * 256; i += 256) h[i] = 0;
  __syncthreads();
  for (int64_t i = (int64_t)blockIdx.x * 256 + threadIdx.x; i < n; i += (int64_t)gridDim.x * 256) {
    const K k = keys[i];
    for (int p = 0; p < passes; ++p) atomicAdd(&h[p * 256 + (int)((k >> (begin_bit + 8 * p)) & 255)], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < passes * 256; i += 256)
    if (h[i]) atomicAdd(&hist[i], h[i]);
}

// sum of the predecessors' values up to (and including) the nearest tile that published its
// inclusive prefix: kSortWindow words read together per round trip, newest first
__device__ __forceinline__ unsigned long long sort_lookback(const unsigned long long* status, int64_t t, int stride,
                                                            int slot, unsigned long long tag) {
  unsigned long long excl = 0;
  int64_t q = t - 1;
  while (q >= 0) {
    unsigned long long w[kSortWindow];
#pragma unroll
    for (int j = 0; j < kSortWindow; ++j) w[j] = q - j >= 0 ? ld_relaxed(status + (q - j) * stride + slot) : 0ull;
    int j = 0;
    for (; j < kSortWindow && q - j >= 0; ++j) {
      unsigned long long v = w[j];
      while ((v & ~((1ull << 48) - 1)) != tag || ((v >> 46) & 3ull) == 0) v = ld_relaxed(status + (q - j) * stride + slot);
      excl += v & kSortValMask;
      if (((v >> 46) & 3ull) == kSortPre) return excl;
    }
    q -= j;
  }
  return excl;
}

template <typename K, bool VALS>
__global__ void __launch_bounds__(kSortThreads, sizeof(K) == 8 && VALS ? 3 : 4) sort_pass_kernel(const __grid_constant__ SortPass p) {
  __shared__ uint32_t s_wcnt[kSortThreads / 32][256];  // per-warp digit counters, then warp bases
  __shared__ uint32_t s_local[256];                     // tile-local exclusive offset of each digit
  __shared__ unsigned long long s_gbase[256];           // global destination of each digit's first element
  __shared__ unsigned long long s_scan[33];
  __shared__ K s_keys[kSortTile];                       // keys in sorted (digit) order
  __shared__ unsigned long long s_vals[VALS ? kSortTile : 1];  // their values
  __shared__ long long s_tile;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) s_tile = (long long)atomicAdd(p.ticket, 1ull);
  for (int i = threadIdx.x; i < (kSortThreads / 32) * 256; i += kSortThreads) (&s_wcnt[0][0])[i] = 0;
  __syncthreads();
  const int64_t t = s_tile;
  // warp-striped items: element t*T + warp*256 + j*32 + lane (coalesced loads; tile order =
  // (warp, j, lane) = ascending element index, which the ranks below preserve)
  const int64_t e0 = t * kSortTile + (int64_t)warp * (32 * kSortItems);
  const K* kin = static_cast<const K*>(p.keys_in);
  K key[kSortItems];
  unsigned long long val[kSortItems];
  int dig[kSortItems];
  uint32_t rank[kSortItems];
#pragma unroll
  for (int j = 0; j < kSortItems; ++j) {
    const int64_t e = e0 + j * 32 + lane;
    const bool ok = e < p.n;
    key[j] = ok ? kin[e] : (K)0;
    if (VALS) val[j] = ok ? p.vals_in[e] : 0ull;
    dig[j] = ok ? (int)((key[j] >> p.shift) & 255) : 256;
  }
  const uint32_t lt = (1u << lane) - 1u;
#pragma unroll
  for (int j = 0; j < kSortItems; ++j) {  // stable warp-local ranks, item slot by item slot
    const uint32_t peers = __match_any_sync(0xFFFFFFFFu, dig[j]);
    const uint32_t base = dig[j] < 256 ? s_wcnt[warp][dig[j]] : 0u;
    rank[j] = base + __popc(peers & lt);
    __syncwarp();
    if (dig[j] < 256 && (peers & lt) == 0) s_wcnt[warp][dig[j]] = base + __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  const int d = threadIdx.x;  // one thread per digit
  uint32_t tot = 0;
#pragma unroll
  for (int w = 0; w < kSortThreads / 32; ++w) {
    const uint32_t c = s_wcnt[w][d];
    s_wcnt[w][d] = tot;
    tot += c;
  }
  unsigned long long* st = p.status + t * 256;
  st_relaxed(st + d, p.tag | ((t == 0 ? kSortPre : kSortAgg) << 46) | tot);
  unsigned long long tile_n;
  const unsigned long long loc = block_excl_scan(tot, s_scan, &tile_n);
  s_local[d] = (uint32_t)loc;
  unsigned long long g_all;
  const unsigned long long gd = block_excl_scan(p.hist[d], s_scan, &g_all);  // (its barriers publish s_local)
  // the tile-local sort into shared memory BEFORE the look-back: the keys' and values' registers
  // are free while the digit threads wait on their predecessors (no spills at 3-4 blocks per SM)
#pragma unroll
  for (int j = 0; j < kSortItems; ++j) {
    if (dig[j] < 256) {
      const uint32_t pos = s_local[dig[j]] + s_wcnt[warp][dig[j]] + rank[j];
      s_keys[pos] = key[j];
      if (VALS) s_vals[pos] = val[j];
    }
  }
  unsigned long long excl = 0;
  if (t > 0) {
    excl = sort_lookback(p.status, t, 256, d, p.tag);
    st_relaxed(st + d, p.tag | (kSortPre << 46) | (excl + tot));
  }
  s_gbase[d] = gd + excl;
  __syncthreads();
  K* kout = static_cast<K*>(p.keys_out);
  for (int i = threadIdx.x; i < (int)tile_n; i += kSortThreads) {  // runs of one digit: coalesced
    const K k = s_keys[i];
    const int dd = (int)((k >> p.shift) & 255);
    const unsigned long long dst = s_gbase[dd] + (unsigned long long)(i - (int)s_local[dd]);
    kout[dst] = k;
    if (VALS) p.vals_out[dst] = s_vals[i];
  }
}

// ---- runs of sorted keys ------------------------------------------------------------------------
enum { ESC_KEY_RAW = 0, ESC_KEY_U32 = 1, ESC_KEY_I32 = 2, ESC_KEY_I64 = 3 };  // esc_runs key decodings

template <typename K>
__device__ __forceinline__ long long decode_key(K k, int mode) {
  switch (mode) {
    case ESC_KEY_I32: return (long long)(int32_t)((uint32_t)k ^ 0x80000000u);
    case ESC_KEY_I64: return (long long)((unsigned long long)k ^ (1ull << 63));
    default: return (long long)k;
  }
}

struct RunsParams {
  const void* keys;
  int64_t n;
  int32_t decode;
  int32_t pad;
  long long* unique_keys;      // [runs]
  long long* starts;           // [runs + 1]
  long long* run_of;           // [n] or nullptr
  unsigned long long* status;  // [tiles]
  unsigned long long* ticket;
  long long* stats;            // [4]: runs, first key, last key, largest run (set by runs_finish_kernel)
  unsigned long long tag;
};

template <typename K>
__global__ void __launch_bounds__(kSortThreads) runs_kernel(const __grid_constant__ RunsParams p) {
  __shared__ unsigned long long s_scan[33];
  __shared__ long long s_tile;
  __shared__ unsigned long long s_base;
  if (threadIdx.x == 0) s_tile = (long long)atomicAdd(p.ticket, 1ull);
  __syncthreads();
  const int64_t t = s_tile;
  const K* keys = static_cast<const K*>(p.keys);
  const int64_t i0 = t * kSortTile + (int64_t)threadIdx.x * kSortItems;  // blocked: 8 consecutive per thread
  K k[kSortItems];
  int flag[kSortItems];
  int nf = 0;
#pragma unroll
  for (int j = 0; j < kSortItems; ++j) {
    const int64_t i = i0 + j;
    k[j] = i < p.n ? keys[i] : (K)0;
    const K prev = j > 0 ? k[j - 1] : (i > 0 && i - 1 < p.n ? keys[i - 1] : (K)0);
    flag[j] = (i < p.n && (i == 0 || k[j] != prev)) ? 1 : 0;
    nf += flag[j];
  }
  unsigned long long tile_runs;
  const unsigned long long ex = block_excl_scan((unsigned long long)nf, s_scan, &tile_runs);
  if (threadIdx.x == 0) {
    st_relaxed(p.status + t, p.tag | ((t == 0 ? kSortPre : kSortAgg) << 46) | tile_runs);
    unsigned long long b = 0;
    if (t > 0) {
      b = sort_lookback(p.status, t, 1, 0, p.tag);
      st_relaxed(p.status + t, p.tag | (kSortPre << 46) | (b + tile_runs));
    }
    s_base = b;
    const int64_t last = (p.n - 1) / kSortTile;
    if (t == last) {  // the tile holding the last element closes the run list
      p.starts[b + tile_runs] = p.n;
      p.stats[0] = (long long)(b + tile_runs);
    }
  }
  __syncthreads();
  long long g = (long long)(s_base + ex);
#pragma unroll
  for (int j = 0; j < kSortItems; ++j) {
    const int64_t i = i0 + j;
    if (i >= p.n) break;
    if (flag[j]) {
      p.unique_keys[g] = decode_key<K>(k[j], p.decode);
      p.starts[g] = i;
      ++g;
    }
    if (p.run_of != nullptr) p.run_of[i] = g - 1;
  }
}

// run sizes and the statistics (first / last key, largest run)
__global__ void __launch_bounds__(256) runs_finish_kernel(const long long* __restrict__ starts,
                                                          const long long* __restrict__ unique_keys,
                                                          long long* __restrict__ counts, long long* stats) {
  __shared__ unsigned long long s_red[8];
  const long long u = stats[0];
  long long most = 0;
  for (long long g = (long long)blockIdx.x * 256 + threadIdx.x; g < u; g += (long long)gridDim.x * 256) {
    const long long c = starts[g + 1] - starts[g];
    if (counts != nullptr) counts[g] = c;
    most = c > most ? c : most;
  }
#pragma unroll
  for (int dd = 16; dd > 0; dd >>= 1) {
    const long long o = __shfl_xor_sync(0xFFFFFFFFu, most, dd);
    most = o > most ? o : most;
  }
  if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = (unsigned long long)most;
  __syncthreads();
  if (threadIdx.x == 0) {
    long long m = 0;
    for (int w = 0; w < 8; ++w) m = (long long)s_red[w] > m ? (long long)s_red[w] : m;
    atomicMax(reinterpret_cast<unsigned long long*>(stats + 3), (unsigned long long)m);
    if (blockIdx.x == 0) {
      stats[1] = u > 0 ? unique_keys[0] : 0;
      stats[2] = u > 0 ? unique_keys[u - 1] : 0;
    }
  }
}

// ---- helpers of the f3 / f4 users -----------------------------------------------------------
// order-preserving unsigned keys of an integer column: 1-4 byte signed -> u32 ^ 2^31, unsigned ->
// u32, int64 -> u64 ^ 2^63
__global__ void order_keys_kernel(const uint8_t* __restrict__ in, int dtype, int width, int64_t n, void* out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const long long v = ld_int(in + (size_t)i * width, dtype);
    if (width == 8) static_cast<unsigned long long*>(out)[i] = (unsigned long long)v ^ (1ull << 63);
    else if (dtype == ESC_U8 || dtype == ESC_U16 || dtype == ESC_U32) static_cast<uint32_t*>(out)[i] = (uint32_t)v;
    else static_cast<uint32_t*>(out)[i] = (uint32_t)(int32_t)v ^ 0x80000000u;
  }
}

// the run holding sorted position pos: the last start <= pos
__device__ __forceinline__ long long run_at(const long long* __restrict__ starts, long long u, long long pos) {
  long long lo = 0, hi = u;  // answer in [0, u)
  while (hi - lo > 1) {
    const long long mid = (lo + hi) >> 1;
    if (starts[mid] <= pos) lo = mid;
    else hi = mid;
  }
  return lo;
}

// values at sorted positions: out[i] = unique_keys[run_at(ranks[i])]
__global__ void rank_values_kernel(const long long* __restrict__ uk, const long long* __restrict__ starts,
                                   const long long* __restrict__ stats, const long long* __restrict__ ranks, int k,
                                   long long* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < k) out[i] = uk[run_at(starts, stats[0], ranks[i])];
}

// equi-depth buckets over a sorted column given as runs: bucket j covers [lo_j, hi_j) with
// hi_j = the end of the last run whose value <= bounds[j+1] (the last bucket ends at n), and
// holds run_at(hi_j - 1) - run_at(lo_j) + 1 distinct values
__global__ void hist_buckets_kernel(const long long* __restrict__ uk, const long long* __restrict__ starts,
                                    const long long* __restrict__ stats, int64_t n, const long long* __restrict__ bounds,
                                    int nb, long long* __restrict__ out_hi, long long* __restrict__ out_distinct) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= nb) return;
  const long long u = stats[0];
  auto hi_of = [&](int b) -> long long {
    if (b == nb - 1) return n;
    const long long v = bounds[b + 1];
    long long lo = 0, hi = u;  // first run with key > v
    while (lo < hi) {
      const long long mid = (lo + hi) >> 1;
      if (uk[mid] <= v) lo = mid + 1;
      else hi = mid;
    }
    return starts[lo];
  };
  const long long hi = hi_of(j);
  const long long lo = j == 0 ? 0 : hi_of(j - 1);
  out_hi[j] = hi;
  out_distinct[j] = hi > lo ? run_at(starts, u, hi - 1) - run_at(starts, u, lo) + 1 : 0;
}

// ---- first-appearance dictionary codes (CSV TEXT columns) -------------------------------------
// sort key of a cell: its 64-bit content hash >> 1, or 2^63 for a NULL (so NULLs are the last run)
__global__ void dict_keys_kernel(const long long* __restrict__ hashes, const uint8_t* __restrict__ nulls, int64_t n,
                                 unsigned long long* __restrict__ keys, unsigned long long* __restrict__ rows) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const bool null = nulls != nullptr && nulls[i];
    keys[i] = null ? (1ull << 63) : ((unsigned long long)hashes[i] >> 1);
    rows[i] = (unsigned long long)i;
  }
}

// per run: its first row (= the row at its start: the sort is stable) as the second sort's key
// (0xFFFFFFFF pads the NULL run and positions past the last run) and the run id as its value
__global__ void dict_firsts_kernel(const long long* __restrict__ starts, const unsigned long long* __restrict__ srows,
                                   const unsigned long long* __restrict__ skeys, const long long* __restrict__ stats,
                                   int64_t n, uint32_t* __restrict__ first_key, unsigned long long* __restrict__ run_id) {
  const long long u = stats[0];
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
    uint32_t k = 0xFFFFFFFFu;
    if (r < u) {
      const long long s = starts[r];
      if (skeys[s] != (1ull << 63)) k = (uint32_t)srows[s];
    }
    first_key[r] = k;
    run_id[r] = (unsigned long long)r;
  }
}

// code of every run = its position in first-appearance order; first row of every code
__global__ void dict_code_of_kernel(const uint32_t* __restrict__ sorted_first, const unsigned long long* __restrict__ sorted_run,
                                    int64_t n, long long* __restrict__ code_of, long long* __restrict__ first_of_code,
                                    long long* __restrict__ n_codes) {
  for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < n; c += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t f = sorted_first[c];
    if (f == 0xFFFFFFFFu) {
      if (c == 0 || sorted_first[c - 1] != 0xFFFFFFFFu) *n_codes = c;  // the first padding position
      continue;
    }
    code_of[sorted_run[c]] = c;
    first_of_code[c] = (long long)f;
    if (c == n - 1) *n_codes = n;
  }
}

// every cell's code and representative row (NULL: code 0, representative -1)
__global__ void dict_scatter_kernel(const unsigned long long* __restrict__ skeys, const unsigned long long* __restrict__ srows,
                                    const long long* __restrict__ run_of, const long long* __restrict__ starts,
                                    const long long* __restrict__ code_of, int64_t n, int32_t* __restrict__ codes,
                                    long long* __restrict__ rep) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const long long row = (long long)srows[i];
    if (skeys[i] == (1ull << 63)) {
      codes[row] = 0;
      rep[row] = -1;
      continue;
    }
    const long long r = run_of[i];
    codes[row] = (int32_t)code_of[r];
    rep[row] = (long long)srows[starts[r]];
  }
}

}  // namespace esc

// ==========================================================================================
// host side
// ==========================================================================================
namespace {

struct SortLayout {
  size_t counters, hist, status, runs_status, keys_alt, vals_alt, total;
  int64_t tiles;
};

// [counters][histograms][status: tiles x 256][runs status: tiles][keys alt][values alt]: every
// region up to keys_alt depends on n only (the same offsets with or without values), and the
// status regions are cleared at the start of each call, so no stale word — a previous call's
// status or any other data the caller's buffer held — can pass for a published one; within a
// call the sort's passes tag their words 1..8
SortLayout sort_layout(int64_t n, int key_bytes, bool vals) {
  SortLayout L;
  auto up = [](size_t x) { return (x + 255) & ~(size_t)255; };
  L.tiles = (n + esc::kSortTile - 1) / esc::kSortTile;
  const size_t tiles = (size_t)(L.tiles > 0 ? L.tiles : 1);
  L.counters = 0;                                               // pass tickets + runs ticket
  L.hist = up(L.counters + 16 * sizeof(unsigned long long));    // passes x 256 u32
  L.status = up(L.hist + esc::kSortMaxPasses * 256 * sizeof(uint32_t));
  L.runs_status = up(L.status + tiles * 256 * 8);
  L.keys_alt = up(L.runs_status + tiles * 8);
  L.vals_alt = up(L.keys_alt + (size_t)n * key_bytes);
  L.total = up(L.vals_alt + (vals ? (size_t)n * 8 : 0));
  return L;
}

template <typename K>
int sort_pairs_t(const K* keys_in, const uint64_t* vals_in, K* keys_out, uint64_t* vals_out, int64_t n, int begin_bit,
                 int end_bit, uint8_t* temp, const SortLayout& L, cudaStream_t st) {
  const int passes = (end_bit - begin_bit + 7) / 8;
  cudaError_t e = cudaMemsetAsync(temp, 0, L.runs_status, st);  // tickets, histograms, status words
  if (e != cudaSuccess) return fail(ESC_ERR_CUDA, std::string("sort init: ") + cudaGetErrorString(e));
  uint32_t* hist = reinterpret_cast<uint32_t*>(temp + L.hist);
  const int sms = sm_count_cached();
  if (sms <= 0) return fail(ESC_ERR_CUDA, "no CUDA device");
  int64_t hb = (n + 255) / 256;
  if (hb > (int64_t)sms * 4) hb = (int64_t)sms * 4;
  ++g_launches;
  esc::sort_hist_kernel<K><<<(unsigned)hb, 256, 0, st>>>(keys_in, n, begin_bit, passes, hist);
  K* alt = reinterpret_cast<K*>(temp + L.keys_alt);
  uint64_t* valt = reinterpret_cast<uint64_t*>(temp + L.vals_alt);
  const K* src = keys_in;
  const uint64_t* vsrc = vals_in;
  for (int p = 0; p < passes; ++p) {
    const uint32_t tag = (uint32_t)p + 1;
    const bool to_out = ((passes - 1 - p) % 2) == 0;  // the last pass lands in keys_out
    esc::SortPass sp;
    sp.keys_in = src;
    sp.vals_in = reinterpret_cast<const unsigned long long*>(vsrc);
    sp.keys_out = to_out ? keys_out : alt;
    sp.vals_out = reinterpret_cast<unsigned long long*>(vals_in != nullptr ? (to_out ? vals_out : valt) : nullptr);
    sp.n = n;
    sp.shift = begin_bit + 8 * p;
    sp.pad = 0;
    sp.hist = hist + 256 * p;
    sp.status = reinterpret_cast<unsigned long long*>(temp + L.status);
    sp.ticket = reinterpret_cast<unsigned long long*>(temp + L.counters) + p;
    sp.tag = (unsigned long long)tag << 48;
    ++g_launches;
    if (vals_in != nullptr) esc::sort_pass_kernel<K, true><<<(unsigned)L.tiles, esc::kSortThreads, 0, st>>>(sp);
    else esc::sort_pass_kernel<K, false><<<(unsigned)L.tiles, esc::kSortThreads, 0, st>>>(sp);
    src = static_cast<const K*>(sp.keys_out);
    vsrc = reinterpret_cast<const uint64_t*>(sp.vals_out);
  }
  e = cudaGetLastError();
  if (e != cudaSuccess) return fail(ESC_ERR_CUDA, std::string("sort launch: ") + cudaGetErrorString(e));
  return ESC_OK;
}

template <typename K>
int runs_t(const K* keys, int64_t n, int decode, long long* unique_keys, long long* starts, long long* counts,
           long long* run_of, long long* stats, uint8_t* temp, const SortLayout& L, cudaStream_t st) {
  cudaError_t e = cudaMemsetAsync(stats, 0, 4 * sizeof(long long), st);
  if (e == cudaSuccess) e = cudaMemsetAsync(temp + L.counters + 15 * 8, 0, 8, st);  // the runs ticket
  if (e == cudaSuccess) e = cudaMemsetAsync(temp + L.runs_status, 0, (size_t)(L.tiles > 0 ? L.tiles : 1) * 8, st);
  if (e == cudaSuccess && n == 0) e = cudaMemsetAsync(starts, 0, sizeof(long long), st);
  if (e != cudaSuccess) return fail(ESC_ERR_CUDA, std::string("runs init: ") + cudaGetErrorString(e));
  if (n == 0) return ESC_OK;
  const uint32_t tag = 1;
  esc::RunsParams rp;
  rp.keys = keys;
  rp.n = n;
  rp.decode = decode;
  rp.pad = 0;
  rp.unique_keys = unique_keys;
  rp.starts = starts;
  rp.run_of = run_of;
  rp.status = reinterpret_cast<unsigned long long*>(temp + L.runs_status);
  rp.ticket = reinterpret_cast<unsigned long long*>(temp + L.counters) + 15;
  rp.stats = stats;
  rp.tag = (unsigned long long)tag << 48;
  g_launches += 2;
  esc::runs_kernel<K><<<(unsigned)L.tiles, esc::kSortThreads, 0, st>>>(rp);
  const int sms = sm_count_cached();
  int64_t fb = (n + 255) / 256;
  if (fb > (int64_t)sms * 4) fb = (int64_t)sms * 4;
  esc::runs_finish_kernel<<<(unsigned)(fb > 0 ? fb : 1), 256, 0, st>>>(starts, unique_keys, counts, stats);
  e = cudaGetLastError();
  if (e != cudaSuccess) return fail(ESC_ERR_CUDA, std::string("runs launch: ") + cudaGetErrorString(e));
  return ESC_OK;
}

}  // namespace

extern "C" {

size_t esc_sort_temp_bytes(int64_t n, int32_t key_bytes, int32_t with_values) {
  if (n < 0 || (key_bytes != 4 && key_bytes != 8)) return 0;
  return sort_layout(n, key_bytes, with_values != 0).total;
}

int esc_sort_pairs(const void* keys_in, const uint64_t* vals_in, void* keys_out, uint64_t* vals_out, int64_t n,
                   int32_t key_bytes, int32_t begin_bit, int32_t end_bit, void* temp, size_t temp_bytes,
                   void* stream) {
  if (n < 0 || n >= (1ll << 40) || (key_bytes != 4 && key_bytes != 8))
    return fail(ESC_ERR_INVALID, "bad sort size / key width");
  if (begin_bit < 0 || end_bit > key_bytes * 8 || begin_bit >= end_bit || (end_bit - begin_bit) > 64)
    return fail(ESC_ERR_INVALID, "bad sort bit range");
  if (n == 0) return ESC_OK;
  if (keys_in == nullptr || keys_out == nullptr || temp == nullptr || (vals_in != nullptr && vals_out == nullptr))
    return fail(ESC_ERR_INVALID, "null sort buffer");
  const SortLayout L = sort_layout(n, key_bytes, vals_in != nullptr);
  if (temp_bytes < L.total) return fail(ESC_ERR_WORKSPACE, "sort temp too small");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (key_bytes == 4)
    return sort_pairs_t<uint32_t>(static_cast<const uint32_t*>(keys_in), vals_in, static_cast<uint32_t*>(keys_out),
                                  vals_out, n, begin_bit, end_bit, static_cast<uint8_t*>(temp), L, st);
  return sort_pairs_t<unsigned long long>(static_cast<const unsigned long long*>(keys_in), vals_in,
                                          static_cast<unsigned long long*>(keys_out), vals_out, n, begin_bit, end_bit,
                                          static_cast<uint8_t*>(temp), L, st);
}

int esc_runs(const void* sorted_keys, int32_t key_bytes, int32_t decode, int64_t n, int64_t* unique_keys,
             int64_t* starts, int64_t* counts, int64_t* run_of, int64_t* stats, void* temp, size_t temp_bytes,
             void* stream) {
  if (n < 0 || n >= (1ll << 40) || (key_bytes != 4 && key_bytes != 8) || decode < 0 || decode > 3)
    return fail(ESC_ERR_INVALID, "bad runs arguments");
  if (stats == nullptr || starts == nullptr || temp == nullptr || (n > 0 && (sorted_keys == nullptr || unique_keys == nullptr)))
    return fail(ESC_ERR_INVALID, "null runs buffer");
  const SortLayout L = sort_layout(n, key_bytes, false);
  if (temp_bytes < L.total) return fail(ESC_ERR_WORKSPACE, "runs temp too small");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  uint8_t* t = static_cast<uint8_t*>(temp);
  long long* uk = reinterpret_cast<long long*>(unique_keys);
  long long* s = reinterpret_cast<long long*>(starts);
  long long* c = reinterpret_cast<long long*>(counts);
  long long* r = reinterpret_cast<long long*>(run_of);
  long long* sts = reinterpret_cast<long long*>(stats);
  if (key_bytes == 4) return runs_t<uint32_t>(static_cast<const uint32_t*>(sorted_keys), n, decode, uk, s, c, r, sts, t, L, st);
  return runs_t<unsigned long long>(static_cast<const unsigned long long*>(sorted_keys), n, decode, uk, s, c, r, sts, t,
                                    L, st);
}

int esc_order_keys(const void* values, int32_t dtype, int64_t n, void* out, void* stream) {
  const int w = dtype_width(dtype);
  if (w == 0 || dtype == ESC_F32 || dtype == ESC_F64) return fail(ESC_ERR_UNSUPPORTED, "sort keys must be integers");
  if (n < 0 || (n > 0 && (values == nullptr || out == nullptr))) return fail(ESC_ERR_INVALID, "bad key arguments");
  if (n == 0) return ESC_OK;
  const int sms = sm_count_cached();
  int64_t blocks = (n + 255) / 256;
  if (blocks > (int64_t)sms * 8) blocks = (int64_t)sms * 8;
  ++g_launches;
  esc::order_keys_kernel<<<(unsigned)blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const uint8_t*>(values), dtype, w, n, out);
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? ESC_OK : fail(ESC_ERR_CUDA, std::string("order keys: ") + cudaGetErrorString(e));
}

int esc_rank_values(const int64_t* unique_keys, const int64_t* starts, const int64_t* stats, const int64_t* ranks,
                    int32_t k, int64_t* out, void* stream) {
  if (k < 0 || (k > 0 && (unique_keys == nullptr || starts == nullptr || stats == nullptr || ranks == nullptr ||
                          out == nullptr)))
    return fail(ESC_ERR_INVALID, "bad rank arguments");
  if (k == 0) return ESC_OK;
  ++g_launches;
  esc::rank_values_kernel<<<(k + 255) / 256, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      reinterpret_cast<const long long*>(unique_keys), reinterpret_cast<const long long*>(starts),
      reinterpret_cast<const long long*>(stats), reinterpret_cast<const long long*>(ranks), k,
      reinterpret_cast<long long*>(out));
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? ESC_OK : fail(ESC_ERR_CUDA, std::string("rank values: ") + cudaGetErrorString(e));
}

int esc_hist_buckets(const int64_t* unique_keys, const int64_t* starts, const int64_t* stats, int64_t n,
                     const int64_t* bounds, int32_t nb, int64_t* out_hi, int64_t* out_distinct, void* stream) {
  if (nb < 0 || (nb > 0 && (unique_keys == nullptr || starts == nullptr || stats == nullptr || bounds == nullptr ||
                            out_hi == nullptr || out_distinct == nullptr)))
    return fail(ESC_ERR_INVALID, "bad bucket arguments");
  if (nb == 0) return ESC_OK;
  ++g_launches;
  esc::hist_buckets_kernel<<<(nb + 255) / 256, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      reinterpret_cast<const long long*>(unique_keys), reinterpret_cast<const long long*>(starts),
      reinterpret_cast<const long long*>(stats), n, reinterpret_cast<const long long*>(bounds), nb,
      reinterpret_cast<long long*>(out_hi), reinterpret_cast<long long*>(out_distinct));
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? ESC_OK : fail(ESC_ERR_CUDA, std::string("histogram buckets: ") + cudaGetErrorString(e));
}

namespace {
struct DictLayout {
  size_t keys, rows, skeys, srows, uk, starts, run_of, first_key, run_id, sfirst, srun, code_of, stats, sort, total;
};
DictLayout dict_layout(int64_t n) {
  DictLayout L;
  auto up = [](size_t x) { return (x + 255) & ~(size_t)255; };
  const size_t w = (size_t)(n > 0 ? n : 1) * 8;
  size_t o = 0;
  L.keys = o; o = up(o + w);
  L.rows = o; o = up(o + w);
  L.skeys = o; o = up(o + w);
  L.srows = o; o = up(o + w);
  L.uk = o; o = up(o + w);
  L.starts = o; o = up(o + w + 8);
  L.run_of = o; o = up(o + w);
  L.first_key = o; o = up(o + w);
  L.run_id = o; o = up(o + w);
  L.sfirst = o; o = up(o + w);
  L.srun = o; o = up(o + w);
  L.code_of = o; o = up(o + w);
  L.stats = o; o = up(o + 64);
  L.sort = o; o = up(o + sort_layout(n, 8, true).total);
  L.total = o;
  return L;
}
}  // namespace

size_t esc_dict_temp_bytes(int64_t n) { return n < 0 ? 0 : dict_layout(n).total; }

int esc_dict_encode(const int64_t* hashes, const uint8_t* nulls, int64_t n, int32_t* out_codes, int64_t* out_rep,
                    int64_t* out_first, int64_t* out_n_codes, void* temp, size_t temp_bytes, void* stream) {
  if (n < 0 || n >= (1ll << 31)) return fail(ESC_ERR_INVALID, "bad dictionary size");
  if (out_n_codes == nullptr || (n > 0 && (hashes == nullptr || out_codes == nullptr || out_rep == nullptr ||
                                           out_first == nullptr || temp == nullptr)))
    return fail(ESC_ERR_INVALID, "null dictionary buffer");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (n == 0) {
    const cudaError_t e = cudaMemsetAsync(out_n_codes, 0, 8, st);
    return e == cudaSuccess ? ESC_OK : fail(ESC_ERR_CUDA, std::string("dictionary init: ") + cudaGetErrorString(e));
  }
  const DictLayout L = dict_layout(n);
  if (temp_bytes < L.total) return fail(ESC_ERR_WORKSPACE, "dictionary temp too small");
  uint8_t* t = static_cast<uint8_t*>(temp);
  auto u64 = [&](size_t off) { return reinterpret_cast<unsigned long long*>(t + off); };
  auto i64 = [&](size_t off) { return reinterpret_cast<long long*>(t + off); };
  const size_t sort_bytes = sort_layout(n, 8, true).total;
  const int sms = sm_count_cached();
  int64_t blocks = (n + 255) / 256;
  if (blocks > (int64_t)sms * 8) blocks = (int64_t)sms * 8;
  ++g_launches;
  esc::dict_keys_kernel<<<(unsigned)blocks, 256, 0, st>>>(reinterpret_cast<const long long*>(hashes), nulls, n,
                                                          u64(L.keys), u64(L.rows));
  // cells grouped by content hash, each group in row order (stable), NULLs last
  int rc = esc_sort_pairs(u64(L.keys), reinterpret_cast<const uint64_t*>(u64(L.rows)), u64(L.skeys),
                          reinterpret_cast<uint64_t*>(u64(L.srows)), n, 8, 0, 64, t + L.sort, sort_bytes, st);
  if (rc == ESC_OK)
    rc = esc_runs(u64(L.skeys), 8, esc::ESC_KEY_RAW, n, reinterpret_cast<int64_t*>(i64(L.uk)),
                  reinterpret_cast<int64_t*>(i64(L.starts)), nullptr, reinterpret_cast<int64_t*>(i64(L.run_of)),
                  reinterpret_cast<int64_t*>(i64(L.stats)), t + L.sort, sort_bytes, st);
  if (rc != ESC_OK) return rc;
  g_launches += 3;
  esc::dict_firsts_kernel<<<(unsigned)blocks, 256, 0, st>>>(i64(L.starts), u64(L.srows), u64(L.skeys), i64(L.stats),
                                                            n, reinterpret_cast<uint32_t*>(t + L.first_key),
                                                            u64(L.run_id));
  // runs in first-appearance order (first rows < 2^31: 4 digit passes; padding sorts last)
  rc = esc_sort_pairs(t + L.first_key, reinterpret_cast<const uint64_t*>(u64(L.run_id)), t + L.sfirst,
                      reinterpret_cast<uint64_t*>(u64(L.srun)), n, 4, 0, 32, t + L.sort, sort_bytes, st);
  if (rc != ESC_OK) return rc;
  esc::dict_code_of_kernel<<<(unsigned)blocks, 256, 0, st>>>(reinterpret_cast<const uint32_t*>(t + L.sfirst),
                                                             u64(L.srun), n, i64(L.code_of),
                                                             reinterpret_cast<long long*>(out_first),
                                                             reinterpret_cast<long long*>(out_n_codes));
  esc::dict_scatter_kernel<<<(unsigned)blocks, 256, 0, st>>>(u64(L.skeys), u64(L.srows), i64(L.run_of),
                                                             i64(L.starts), i64(L.code_of), n, out_codes,
                                                             reinterpret_cast<long long*>(out_rep));
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? ESC_OK : fail(ESC_ERR_CUDA, std::string("dictionary encode: ") + cudaGetErrorString(e));
}

}  // extern "C"
