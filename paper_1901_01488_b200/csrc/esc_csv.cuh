// esc_csv.cuh — CSV ingestion into device columns, included by esc_kernels.cu.
//
// Replaces storage.load_csv / append_rows' cell conversion (storage.py:245-275, :385-409): the
// file's bytes are copied to HBM once and tokenised, validated and converted there, so a table
// never crosses PCIe again (the columns stay resident for every ESC sub-query).
//
//   pass 1  esc_csv_count   per 16 KB chunk and per 1 KB warp slice (16 bytes per lane, one
//                           16-byte load each): quote parity and the
//                           separators / record ends outside quotes for BOTH possible starting
//                           quote states (composable summaries), then one block scans the chunk
//                           summaries: every chunk's starting state, field and record offsets.
//   pass 2  esc_csv_fields  every separator outside quotes -> field_end[i] (byte position) and
//                           its kind (',', '\n' / lone '\r', "\r\n"), record ends -> rec_end.
//   pass 3  esc_csv_parse   one thread per record and column: field bytes -> int64 value + NULL
//                           flag (INT64 / DECIMAL(p,s) / DATE) or a 64-bit content hash + length
//                           (TEXT, dictionary-encoded by first appearance on the host side); the
//                           first failing cell (row-major, the reference's order) via atomicMin.
//
// Quote state by prefix parity is exact for RFC-4180 fields (quotes only around a field, ""
// inside); any other quote placement is reported as a malformed cell, never mis-split silently.
#pragma once

namespace esc {

constexpr int kCsvChunk = 16384;   // bytes per block
constexpr int kCsvWarps = 16;      // 1 KB slice per warp
constexpr int kCsvSlice = kCsvChunk / kCsvWarps;

// composable summary of a byte range: quote parity flip, separators/record ends outside quotes
// assuming the range starts outside (e) or inside (o) quotes
struct CsvSum {
  unsigned long long flip;
  unsigned long long f_e, f_o;   // field separators
  unsigned long long r_e, r_o;   // record ends
};
__device__ __forceinline__ CsvSum csv_combine(const CsvSum& a, const CsvSum& b) {
  CsvSum c;
  c.flip = a.flip ^ b.flip;
  c.f_e = a.f_e + (a.flip ? b.f_o : b.f_e);
  c.f_o = a.f_o + (a.flip ? b.f_e : b.f_o);
  c.r_e = a.r_e + (a.flip ? b.r_o : b.r_e);
  c.r_o = a.r_o + (a.flip ? b.r_e : b.r_o);
  return c;
}

// 16 consecutive bytes per lane (one 16-byte load; a warp covers 512 bytes per step): the lane
// walks its bytes with the quote state it inherits from the lanes before it (XOR-scan of their
// quote-count parities via one ballot).
struct CsvLane {
  uint8_t c[16];
  uint8_t prev, next;  // the bytes just before / after the lane's 16 (0 outside the text)
  int real;            // bytes of the text in c (< 16 only at its end)
  int cnt;             // bytes this lane processes (<= real: stops at the slice end)
};

__device__ __forceinline__ void csv_load_lane(const uint8_t* b, int64_t n, int64_t i0, int64_t s1, CsvLane& L) {
  L.real = i0 >= n ? 0 : (i0 + 16 <= n ? 16 : (int)(n - i0));
  if (L.real == 16 && (reinterpret_cast<uintptr_t>(b + i0) & 15) == 0) {
    const uint4 v = __ldg(reinterpret_cast<const uint4*>(b + i0));
    memcpy(L.c, &v, 16);
  } else {
#pragma unroll
    for (int k = 0; k < 16; ++k) L.c[k] = k < L.real ? b[i0 + k] : 0;
  }
  L.prev = (i0 > 0 && i0 <= n) ? b[i0 - 1] : 0;
  L.next = (i0 + 16 < n) ? b[i0 + 16] : 0;
  L.cnt = i0 >= s1 ? 0 : (i0 + L.real > s1 ? (int)(s1 - i0) : L.real);
}

// SWAR classification of a lane's 16 bytes into 16-bit masks (bit k = byte k)
__device__ __forceinline__ uint32_t eq_mask4(uint32_t w, uint32_t pat) {
  const uint32_t e = __vcmpeq4(w, pat);  // 0xFF in every byte equal to the pattern byte
  // the four byte-high bits (7, 15, 23, 31) gathered into bits 28..31 by one multiply: each of
  // them meets exactly one of the shifts 21, 14, 7, 0 that lands it there, without carries
  return ((e & 0x80808080u) * 0x00204081u) >> 28;
}

struct CsvMasks {
  uint32_t quote, sep, rec, cr3, valid;
};

__device__ __forceinline__ CsvMasks csv_masks(const CsvLane& L) {
  uint32_t w[4];
  memcpy(w, L.c, 16);
  uint32_t q = 0, comma = 0, cr = 0, lf = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    q |= eq_mask4(w[i], 0x22222222u) << (4 * i);
    comma |= eq_mask4(w[i], 0x2C2C2C2Cu) << (4 * i);
    cr |= eq_mask4(w[i], 0x0D0D0D0Du) << (4 * i);
    lf |= eq_mask4(w[i], 0x0A0A0A0Au) << (4 * i);
  }
  const uint32_t real = L.real >= 16 ? 0xFFFFu : ((1u << L.real) - 1u);
  q &= real; comma &= real; cr &= real; lf &= real;
  CsvMasks m;
  m.valid = L.cnt >= 16 ? 0xFFFFu : ((1u << L.cnt) - 1u);
  const uint32_t cr_before = (cr << 1) | (L.prev == '\r' ? 1u : 0u);   // byte k-1 is '\r'
  const uint32_t lf_after = (lf >> 1) | (L.next == '\n' ? 0x8000u : 0u);  // byte k+1 is '\n'
  m.quote = q & m.valid;
  m.rec = ((lf & ~cr_before) | cr) & m.valid;  // '\n' not after '\r', every '\r'
  m.cr3 = cr & lf_after & m.valid;             // "\r\n": the '\r' ends the record
  m.sep = (comma & m.valid) | m.rec;
  return m;
}

// bit k = parity of the quotes strictly before byte k (quote state relative to the lane start)
__device__ __forceinline__ uint32_t quote_state(uint32_t q) {
  uint32_t x = q;
  x ^= x << 1;
  x ^= x << 2;
  x ^= x << 4;
  x ^= x << 8;
  return (x << 1) & 0xFFFFu;
}

__device__ CsvSum csv_slice_sum(const uint8_t* b, int64_t n, int64_t s0, int64_t s1, int lane) {
  CsvSum acc = {0, 0, 0, 0, 0};
  const unsigned lt = (1u << lane) - 1u;
  for (int64_t base = s0; base < s1; base += 512) {
    CsvLane L;
    const int64_t i0 = base + 16 * lane;
    csv_load_lane(b, n, i0, s1, L);
    const CsvMasks m = csv_masks(L);
    const unsigned odd = __ballot_sync(0xFFFFFFFFu, __popc(m.quote) & 1);
    const uint32_t inside = quote_state(m.quote) ^ (((acc.flip ^ __popc(odd & lt)) & 1u) ? 0xFFFFu : 0u);
    // per-lane counts relative to the slice start state (the combine step's form), reduced
    // over the warp once per slice
    acc.f_e += __popc(m.sep & ~inside);
    acc.f_o += __popc(m.sep & inside);
    acc.r_e += __popc(m.rec & ~inside);
    acc.r_o += __popc(m.rec & inside);
    acc.flip ^= __popc(odd) & 1u;
  }
  acc.f_e = __reduce_add_sync(0xFFFFFFFFu, (unsigned)acc.f_e);
  acc.f_o = __reduce_add_sync(0xFFFFFFFFu, (unsigned)acc.f_o);
  acc.r_e = __reduce_add_sync(0xFFFFFFFFu, (unsigned)acc.r_e);
  acc.r_o = __reduce_add_sync(0xFFFFFFFFu, (unsigned)acc.r_o);
  return acc;
}

struct CsvChunkOut {  // per chunk after the scan
  unsigned int start_in;   // chunk starts inside quotes
  unsigned long long field0, rec0;
};

__global__ void __launch_bounds__(kCsvWarps * 32) csv_count_kernel(const uint8_t* __restrict__ b, int64_t n,
                                                                   CsvSum* __restrict__ warp_sums,
                                                                   CsvSum* __restrict__ chunk_sums) {
  __shared__ CsvSum ws[kCsvWarps];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t s0 = (int64_t)blockIdx.x * kCsvChunk + (int64_t)warp * kCsvSlice;
  const int64_t s1 = s0 + kCsvSlice < n ? s0 + kCsvSlice : n;
  CsvSum s = {0, 0, 0, 0, 0};
  if (s0 < n) s = csv_slice_sum(b, n, s0, s1, lane);
  if (lane == 0) {
    ws[warp] = s;
    warp_sums[(int64_t)blockIdx.x * kCsvWarps + warp] = s;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    CsvSum c = ws[0];
    for (int w = 1; w < kCsvWarps; ++w) c = csv_combine(c, ws[w]);
    chunk_sums[blockIdx.x] = c;
  }
}

// one block: exclusive scan of the chunk summaries from the file start (outside quotes)
__global__ void __launch_bounds__(1024) csv_scan_kernel(const CsvSum* __restrict__ chunk_sums, int64_t nchunks,
                                                        CsvChunkOut* __restrict__ out, unsigned long long* totals) {
  __shared__ CsvSum part[1024];
  const int t = threadIdx.x;
  const int64_t per = (nchunks + 1023) / 1024;
  const int64_t c0 = t * per, c1 = c0 + per < nchunks ? c0 + per : nchunks;
  CsvSum acc = {0, 0, 0, 0, 0};
  for (int64_t c = c0; c < c1; ++c) acc = csv_combine(acc, chunk_sums[c]);
  part[t] = acc;
  __syncthreads();
  // inclusive scan of the per-thread summaries (Hillis-Steele with the ordered operator)
  for (int d = 1; d < 1024; d <<= 1) {
    CsvSum prev = {0, 0, 0, 0, 0};
    const bool has = t >= d;
    if (has) prev = part[t - d];
    __syncthreads();
    if (has) part[t] = csv_combine(prev, part[t]);
    __syncthreads();
  }
  CsvSum run = {0, 0, 0, 0, 0};
  if (t > 0) run = part[t - 1];
  for (int64_t c = c0; c < c1; ++c) {
    out[c].start_in = run.flip;
    out[c].field0 = run.f_e;  // the file starts outside quotes: the "e" column is the real one
    out[c].rec0 = run.r_e;
    run = csv_combine(run, chunk_sums[c]);
  }
  if (t == 1023) {
    totals[0] = part[1023].f_e;
    totals[1] = part[1023].r_e;
    totals[2] = part[1023].flip;
  }
}

__global__ void __launch_bounds__(kCsvWarps * 32) csv_fields_kernel(const uint8_t* __restrict__ b, int64_t n,
                                                                    const CsvSum* __restrict__ warp_sums,
                                                                    const CsvChunkOut* __restrict__ chunks,
                                                                    long long* __restrict__ field_end,
                                                                    uint8_t* __restrict__ field_kind,
                                                                    long long* __restrict__ rec_end_field) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const CsvChunkOut co = chunks[blockIdx.x];
  // this warp's starting state: the chunk start composed with the earlier slices of the chunk
  unsigned long long in_q = co.start_in;
  unsigned long long fidx = co.field0, ridx = co.rec0;
  for (int w = 0; w < warp; ++w) {
    const CsvSum s = warp_sums[(int64_t)blockIdx.x * kCsvWarps + w];
    fidx += in_q ? s.f_o : s.f_e;
    ridx += in_q ? s.r_o : s.r_e;
    in_q ^= s.flip;
  }
  const int64_t s0 = (int64_t)blockIdx.x * kCsvChunk + (int64_t)warp * kCsvSlice;
  const int64_t s1 = s0 + kCsvSlice < n ? s0 + kCsvSlice : n;
  const unsigned lt = (1u << lane) - 1u;
  for (int64_t base = s0; base < s1; base += 512) {
    CsvLane L;
    const int64_t i0 = base + 16 * lane;
    csv_load_lane(b, n, i0, s1, L);
    const CsvMasks m = csv_masks(L);
    const unsigned odd = __ballot_sync(0xFFFFFFFFu, __popc(m.quote) & 1);
    const uint32_t inside = quote_state(m.quote) ^ (((in_q ^ __popc(odd & lt)) & 1u) ? 0xFFFFu : 0u);
    const uint32_t out_sep = m.sep & ~inside, out_rec = m.rec & ~inside;
    const unsigned ns = __popc(out_sep), nr = __popc(out_rec);
    // exclusive offsets of the lane's separators within the warp's 512 bytes
    unsigned es = ns, er = nr;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const unsigned ts = __shfl_up_sync(0xFFFFFFFFu, es, d);
      const unsigned tr = __shfl_up_sync(0xFFFFFFFFu, er, d);
      if (lane >= d) { es += ts; er += tr; }
    }
    const unsigned tot_s = __shfl_sync(0xFFFFFFFFu, es, 31), tot_r = __shfl_sync(0xFFFFFFFFu, er, 31);
    unsigned long long f = fidx + es - ns, r = ridx + er - nr;
    for (uint32_t mm = out_sep; mm; mm &= mm - 1) {
      const int k = __ffs(mm) - 1;
      const uint32_t bit = 1u << k;
      field_end[f] = i0 + k;
      field_kind[f] = (uint8_t)((out_rec & bit) ? ((m.cr3 & bit) ? 3 : 2) : 1);
      if (out_rec & bit) rec_end_field[r++] = (long long)f;
      ++f;
    }
    fidx += tot_s;
    ridx += tot_r;
    in_q ^= __popc(odd) & 1u;
  }
}

// ---- cell conversion ------------------------------------------------------------------------
enum { CSV_OK = 0, CSV_BAD = 1, CSV_QUOTE = 2, CSV_OVERFLOW = 3 };
enum { CSV_INT64 = 0, CSV_DECIMAL = 1, CSV_DATE = 2, CSV_TEXT = 3 };

struct CsvParse {
  const uint8_t* b;
  const long long* field_end;
  const uint8_t* field_kind;
  long long first_field;   // field index of the first data record's first field
  long long nrows;
  int ncols;
  int col;
  int kind;
  int scale;
  long long* values;       // int64 values (TEXT: content hash)
  long long* lengths;      // TEXT: content length (+ quoted flag in bit 62), else unused
  uint8_t* nulls;
  unsigned long long* first_error;  // (row * ncols + col) << 2 | code, atomicMin
  uint32_t* null_seen;              // set to 1 when any cell is NULL (or nullptr)
};

__device__ __forceinline__ bool csv_space(uint8_t c) {  // str.strip()'s ASCII whitespace
  return c == ' ' || c == '\t' || c == '\n' || c == '\r' || c == 0x0b || c == 0x0c || (c >= 0x1c && c <= 0x1f);
}

// days from 1970-01-01 of a proleptic Gregorian date (civil calendar)
__device__ __forceinline__ long long days_from_civil(long long y, unsigned m, unsigned d) {
  y -= m <= 2;
  const long long era = (y >= 0 ? y : y - 399) / 400;
  const unsigned yoe = (unsigned)(y - era * 400);
  const unsigned doy = (153 * (m + (m > 2 ? -3 : 9)) + 2) / 5 + d - 1;
  const unsigned doe = yoe * 365 + yoe / 4 - yoe / 100 + doy;
  return era * 146097 + (long long)doe - 719468;
}

__device__ int csv_int(const uint8_t* s, long long n, long long* out) {
  long long i = 0, j = n;
  while (i < j && csv_space(s[i])) ++i;
  while (j > i && csv_space(s[j - 1])) --j;
  bool neg = false;
  if (i < j && (s[i] == '+' || s[i] == '-')) { neg = s[i] == '-'; ++i; }
  if (i >= j) return CSV_BAD;
  unsigned long long v = 0;
  bool prev_digit = false, any = false;
  const unsigned long long lim = neg ? 9223372036854775808ull : 9223372036854775807ull;
  for (long long k = i; k < j; ++k) {
    const uint8_t c = s[k];
    if (c == '_') {  // Python int(): single underscores between digits
      if (!prev_digit || k + 1 >= j || s[k + 1] < '0' || s[k + 1] > '9') return CSV_BAD;
      prev_digit = false;
      continue;
    }
    if (c < '0' || c > '9') return CSV_BAD;
    const unsigned d = c - '0';
    if (v > (lim - d) / 10) return CSV_OVERFLOW;
    v = v * 10 + d;
    prev_digit = any = true;
  }
  if (!any) return CSV_BAD;
  *out = neg ? (long long)(0ull - v) : (long long)v;
  return CSV_OK;
}

__device__ int csv_decimal(const uint8_t* s, long long n, int scale, long long* out) {
  long long i = 0, j = n;
  while (i < j && csv_space(s[i])) ++i;
  while (j > i && csv_space(s[j - 1])) --j;
  bool neg = false;
  if (i < j && (s[i] == '+' || s[i] == '-')) { neg = s[i] == '-'; ++i; }
  long long dot = -1;
  for (long long k = i; k < j; ++k)
    if (s[k] == '.') { dot = k; break; }
  const long long we = dot < 0 ? j : dot;   // whole digits [i, we)
  const long long fs = dot < 0 ? j : dot + 1;  // fraction digits [fs, j)
  if (we == i && fs == j) return CSV_BAD;  // no digits at all
  for (long long k = i; k < we; ++k) if (s[k] < '0' || s[k] > '9') return CSV_BAD;
  for (long long k = fs; k < j; ++k) if (s[k] < '0' || s[k] > '9') return CSV_BAD;
  if (j - fs > scale) return CSV_BAD + 8;  // more fraction digits than the scale keeps
  unsigned long long v = 0;
  const unsigned long long lim = neg ? 9223372036854775808ull : 9223372036854775807ull;
  auto push = [&](unsigned d) -> bool {
    if (v > (lim - d) / 10) return false;
    v = v * 10 + d;
    return true;
  };
  for (long long k = i; k < we; ++k) if (!push(s[k] - '0')) return CSV_OVERFLOW;
  for (long long k = fs; k < j; ++k) if (!push(s[k] - '0')) return CSV_OVERFLOW;
  for (long long k = j - fs; k < scale; ++k) if (!push(0)) return CSV_OVERFLOW;
  *out = neg ? (long long)(0ull - v) : (long long)v;
  return CSV_OK;
}

__device__ int csv_date(const uint8_t* s, long long n, long long* out) {
  // date.fromisoformat's calendar forms: YYYY-MM-DD and YYYYMMDD (no surrounding spaces)
  unsigned y = 0, m = 0, d = 0;
  auto dig = [&](long long k) { return s[k] >= '0' && s[k] <= '9'; };
  if (n == 10 && s[4] == '-' && s[7] == '-') {
    for (long long k : {0ll, 1ll, 2ll, 3ll, 5ll, 6ll, 8ll, 9ll}) if (!dig(k)) return CSV_BAD;
    y = (s[0] - '0') * 1000 + (s[1] - '0') * 100 + (s[2] - '0') * 10 + (s[3] - '0');
    m = (s[5] - '0') * 10 + (s[6] - '0');
    d = (s[8] - '0') * 10 + (s[9] - '0');
  } else if (n == 8) {
    for (long long k = 0; k < 8; ++k) if (!dig(k)) return CSV_BAD;
    y = (s[0] - '0') * 1000 + (s[1] - '0') * 100 + (s[2] - '0') * 10 + (s[3] - '0');
    m = (s[4] - '0') * 10 + (s[5] - '0');
    d = (s[6] - '0') * 10 + (s[7] - '0');
  } else {
    return CSV_BAD;
  }
  if (y < 1 || m < 1 || m > 12 || d < 1) return CSV_BAD;
  const unsigned mdays[12] = {31, 28, 31, 30, 31, 30, 31, 31, 30, 31, 30, 31};
  const bool leap = (y % 4 == 0 && y % 100 != 0) || y % 400 == 0;
  if (d > mdays[m - 1] + (m == 2 && leap ? 1u : 0u)) return CSV_BAD;
  *out = days_from_civil(y, m, d);
  return CSV_OK;
}

// FNV-1a 64 over the unescaped content
__device__ __forceinline__ unsigned long long fnv_step(unsigned long long h, uint8_t c) {
  return (h ^ c) * 0x100000001B3ull;
}

__global__ void csv_parse_kernel(const CsvParse p) {
  bool seen = false;  // this thread parsed a NULL cell (one store per thread at the end)
  for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < p.nrows;
       r += (long long)gridDim.x * blockDim.x) {
    const long long f = p.first_field + r * p.ncols + p.col;
    const long long start = f == 0 ? 0 : p.field_end[f - 1] + (p.field_kind[f - 1] == 3 ? 2 : 1);
    const long long end = p.field_end[f];
    const uint8_t* s = p.b + start;
    const long long len = end - start;
    int err = CSV_OK;
    long long val = 0;
    bool null_cell = false;
    // unquote: a quoted field is "..." with doubled quotes inside; unquoted fields hold no quote
    bool quoted = len > 0 && s[0] == '"';
    long long clen = len;  // content length after unquoting
    if (quoted) {
      if (len < 2 || s[len - 1] != '"') err = CSV_QUOTE;
      long long k = 1, cl = 0;
      while (err == CSV_OK && k < len - 1) {
        if (s[k] == '"') {
          if (k + 1 < len - 1 && s[k + 1] == '"') { k += 2; ++cl; continue; }
          err = CSV_QUOTE;
          break;
        }
        ++k;
        ++cl;
      }
      clen = cl;
    } else {
      for (long long k = 0; k < len; ++k)
        if (s[k] == '"') { err = CSV_QUOTE; break; }
    }
    // content as one byte range; an escaped quote inside can only be TEXT (no number, date or
    // NULL token holds a '"')
    const uint8_t* c = quoted ? s + 1 : s;
    if (err == CSV_OK && quoted && clen != len - 2 && p.kind != CSV_TEXT) err = CSV_BAD;
    if (err == CSV_OK) {
      null_cell = clen == 2 && c[0] == '\\' && c[1] == 'N';
      if (!null_cell) {
        switch (p.kind) {
          case CSV_INT64: err = csv_int(c, clen, &val); break;
          case CSV_DECIMAL: err = csv_decimal(c, clen, p.scale, &val); break;
          case CSV_DATE: err = csv_date(c, clen, &val); break;
          default: {
            unsigned long long h = 0xCBF29CE484222325ull;
            if (quoted) {
              long long k = 1;
              while (k < len - 1) { h = fnv_step(h, s[k]); k += (s[k] == '"') ? 2 : 1; }
            } else {
              for (long long k = 0; k < len; ++k) h = fnv_step(h, s[k]);
            }
            val = (long long)h;
            p.lengths[r] = clen;
            break;
          }
        }
      }
    }
    if (err != CSV_OK) {
      atomicMin(p.first_error, ((unsigned long long)(r * p.ncols + p.col) << 4) | (unsigned long long)err);
      val = 0;
    }
    p.values[r] = null_cell ? 0 : val;
    p.nulls[r] = null_cell ? 1 : 0;
    seen = seen || null_cell;
  }
  if (seen && p.null_seen != nullptr) *p.null_seen = 1u;
}

// TEXT dictionary check: every cell's content equals its group representative's (no 64-bit hash
// collision); mismatch -> *bad = 1
struct CsvVerify {
  const uint8_t* b;
  const long long* field_end;
  const uint8_t* field_kind;
  long long first_field;
  long long nrows;
  int ncols;
  int col;
  const long long* rep;     // representative row per row (-1: NULL)
  unsigned int* bad;
};

// a field's content bytes in order (quoted: between the quotes, "" read as one quote)
struct CsvCursor {
  const uint8_t* s;
  long long k, end;
  __device__ CsvCursor(const uint8_t* b, const CsvVerify& p, long long r) {
    const long long f = p.first_field + r * p.ncols + p.col;
    const long long st = f == 0 ? 0 : p.field_end[f - 1] + (p.field_kind[f - 1] == 3 ? 2 : 1);
    const long long ln = p.field_end[f] - st;
    s = b + st;
    const bool quoted = ln >= 2 && s[0] == '"';
    k = quoted ? 1 : 0;
    end = quoted ? ln - 1 : ln;
  }
  __device__ bool next(uint8_t* c) {
    if (k >= end) return false;
    *c = s[k];
    k += (s[k] == '"') ? 2 : 1;  // only a doubled quote can occur inside a quoted field
    return true;
  }
};

__global__ void csv_verify_kernel(const CsvVerify p) {
  for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < p.nrows;
       r += (long long)gridDim.x * blockDim.x) {
    const long long q = p.rep[r];
    if (q < 0 || q == r) continue;
    CsvCursor a(p.b, p, r), b(p.b, p, q);
    bool same = true;
    while (same) {
      uint8_t x = 0, y = 0;
      const bool ha = a.next(&x), hb = b.next(&y);
      if (ha != hb) same = false;
      else if (!ha) break;
      else same = x == y;
    }
    if (!same) atomicOr(p.bad, 1u);
  }
}

// ---- record validation (the reference's csv.reader + field-count check, storage.py:247-275) ---
// out[0] = min over bad records of (record << 32 | fields it holds) — a record holds ncols fields,
//          an empty line holds 0 — or ~0 when every record is well formed;
// out[1] = the first field-ending '\r' that is not the last byte (Python's csv rejects a lone CR
//          inside a line), or ~0
struct CsvCheck {
  const uint8_t* b;
  int64_t n;
  const long long* field_end;
  const uint8_t* field_kind;
  int64_t nsep;
  const long long* rec_end;  // the data records (the header's already skipped)
  int64_t nrows;
  long long first_field;
  int32_t ncols;
  unsigned long long* out;
};

__global__ void csv_check_kernel(const CsvCheck p) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < p.nrows; i += stride) {
    const long long e = p.rec_end[i];
    const long long pv = i == 0 ? p.first_field - 1 : p.rec_end[i - 1];
    const long long nf = e - pv;
    const long long start = pv >= 0 ? p.field_end[pv] + (p.field_kind[pv] == 3 ? 2 : 1) : 0;
    const long long got = (nf == 1 && p.field_end[e] == start) ? 0 : nf;
    if (got != p.ncols) atomicMin(p.out, ((unsigned long long)i << 32) | (unsigned long long)(got & 0xFFFFFFFFll));
  }
  for (int64_t f = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; f < p.nsep; f += stride) {
    if (p.field_kind[f] != 2) continue;
    const long long pos = p.field_end[f];
    if (pos < p.n - 1 && p.b[pos] == 13) atomicMin(p.out + 1, (unsigned long long)pos);
  }
}

}  // namespace esc

// ==========================================================================================
// C ABI (CSV ingestion)
// ==========================================================================================
extern "C" {

size_t esc_csv_workspace_bytes(int64_t nbytes) {
  const int64_t chunks = (nbytes + esc::kCsvChunk - 1) / esc::kCsvChunk + 1;
  return (size_t)chunks * (esc::kCsvWarps + 1) * sizeof(esc::CsvSum) + (size_t)chunks * sizeof(esc::CsvChunkOut) +
         64;
}

int esc_csv_count(const uint8_t* d_bytes, int64_t nbytes, uint64_t* d_totals, void* d_ws, size_t ws_bytes,
                  void* stream) {
  if (nbytes < 0 || (nbytes > 0 && d_bytes == nullptr) || d_totals == nullptr) return fail(ESC_ERR_INVALID, "bad CSV arguments");
  if (d_ws == nullptr || ws_bytes < esc_csv_workspace_bytes(nbytes)) return fail(ESC_ERR_WORKSPACE, "CSV workspace too small");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t chunks = (nbytes + esc::kCsvChunk - 1) / esc::kCsvChunk;
  esc::CsvSum* warp_sums = static_cast<esc::CsvSum*>(d_ws);
  esc::CsvSum* chunk_sums = warp_sums + (chunks + 1) * esc::kCsvWarps;
  esc::CsvChunkOut* outs = reinterpret_cast<esc::CsvChunkOut*>(chunk_sums + chunks + 1);
  if (chunks == 0) {
    cudaError_t e = cudaMemsetAsync(d_totals, 0, 3 * sizeof(uint64_t), st);
    return e == cudaSuccess ? ESC_OK : fail(ESC_ERR_CUDA, cudaGetErrorString(e));
  }
  ++g_launches;
  esc::csv_count_kernel<<<(unsigned)chunks, esc::kCsvWarps * 32, 0, st>>>(d_bytes, nbytes, warp_sums, chunk_sums);
  ++g_launches;
  esc::csv_scan_kernel<<<1, 1024, 0, st>>>(chunk_sums, chunks, outs, reinterpret_cast<unsigned long long*>(d_totals));
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(ESC_ERR_CUDA, std::string("CSV count launch: ") + cudaGetErrorString(e));
  return ESC_OK;
}

int esc_csv_fields(const uint8_t* d_bytes, int64_t nbytes, int64_t* d_field_end, uint8_t* d_field_kind,
                   int64_t* d_rec_end_field, void* d_ws, size_t ws_bytes, void* stream) {
  if (nbytes < 0 || (nbytes > 0 && (d_bytes == nullptr || d_field_end == nullptr || d_field_kind == nullptr ||
                                    d_rec_end_field == nullptr)))
    return fail(ESC_ERR_INVALID, "bad CSV arguments");
  if (d_ws == nullptr || ws_bytes < esc_csv_workspace_bytes(nbytes)) return fail(ESC_ERR_WORKSPACE, "CSV workspace too small");
  const int64_t chunks = (nbytes + esc::kCsvChunk - 1) / esc::kCsvChunk;
  if (chunks == 0) return ESC_OK;
  esc::CsvSum* warp_sums = static_cast<esc::CsvSum*>(d_ws);
  esc::CsvSum* chunk_sums = warp_sums + (chunks + 1) * esc::kCsvWarps;
  esc::CsvChunkOut* outs = reinterpret_cast<esc::CsvChunkOut*>(chunk_sums + chunks + 1);
  ++g_launches;
  esc::csv_fields_kernel<<<(unsigned)chunks, esc::kCsvWarps * 32, 0, static_cast<cudaStream_t>(stream)>>>(
      d_bytes, nbytes, warp_sums, outs, reinterpret_cast<long long*>(d_field_end), d_field_kind,
      reinterpret_cast<long long*>(d_rec_end_field));
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(ESC_ERR_CUDA, std::string("CSV fields launch: ") + cudaGetErrorString(e));
  return ESC_OK;
}

int esc_csv_parse(const uint8_t* d_bytes, const int64_t* d_field_end, const uint8_t* d_field_kind, int64_t first_field,
                  int64_t nrows, int32_t ncols, int32_t col, int32_t kind, int32_t scale, int64_t* d_values,
                  int64_t* d_lengths, uint8_t* d_nulls, uint64_t* d_first_error, uint32_t* d_null_seen,
                  void* stream) {
  if (nrows < 0 || ncols <= 0 || col < 0 || col >= ncols || kind < ESC_CSV_INT64 || kind > ESC_CSV_TEXT || scale < 0 || scale > 18)
    return fail(ESC_ERR_INVALID, "bad CSV parse arguments");
  if (nrows == 0) return ESC_OK;
  if (d_bytes == nullptr || d_field_end == nullptr || d_field_kind == nullptr || d_values == nullptr ||
      d_nulls == nullptr || d_first_error == nullptr || (kind == ESC_CSV_TEXT && d_lengths == nullptr))
    return fail(ESC_ERR_INVALID, "null CSV parse buffers");
  esc::CsvParse p;
  p.b = d_bytes;
  p.field_end = reinterpret_cast<const long long*>(d_field_end);
  p.field_kind = d_field_kind;
  p.first_field = first_field;
  p.nrows = nrows;
  p.ncols = ncols;
  p.col = col;
  p.kind = kind;
  p.scale = scale;
  p.values = reinterpret_cast<long long*>(d_values);
  p.lengths = reinterpret_cast<long long*>(d_lengths);
  p.nulls = d_nulls;
  p.first_error = reinterpret_cast<unsigned long long*>(d_first_error);
  p.null_seen = d_null_seen;
  const int sms = sm_count_cached();
  if (sms <= 0) return fail(ESC_ERR_CUDA, "no CUDA device");
  int64_t blocks = (nrows + 255) / 256;
  if (blocks > (int64_t)sms * 16) blocks = (int64_t)sms * 16;
  ++g_launches;
  esc::csv_parse_kernel<<<(unsigned)blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(p);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(ESC_ERR_CUDA, std::string("CSV parse launch: ") + cudaGetErrorString(e));
  return ESC_OK;
}

int esc_csv_verify_text(const uint8_t* d_bytes, const int64_t* d_field_end, const uint8_t* d_field_kind,
                        int64_t first_field, int64_t nrows, int32_t ncols, int32_t col, const int64_t* d_rep,
                        uint32_t* d_bad, void* stream) {
  if (nrows < 0 || ncols <= 0 || col < 0 || col >= ncols) return fail(ESC_ERR_INVALID, "bad CSV verify arguments");
  if (nrows == 0) return ESC_OK;
  esc::CsvVerify p;
  p.b = d_bytes;
  p.field_end = reinterpret_cast<const long long*>(d_field_end);
  p.field_kind = d_field_kind;
  p.first_field = first_field;
  p.nrows = nrows;
  p.ncols = ncols;
  p.col = col;
  p.rep = reinterpret_cast<const long long*>(d_rep);
  p.bad = d_bad;
  const int sms = sm_count_cached();
  if (sms <= 0) return fail(ESC_ERR_CUDA, "no CUDA device");
  int64_t blocks = (nrows + 255) / 256;
  if (blocks > (int64_t)sms * 16) blocks = (int64_t)sms * 16;
  ++g_launches;
  esc::csv_verify_kernel<<<(unsigned)blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(p);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(ESC_ERR_CUDA, std::string("CSV verify launch: ") + cudaGetErrorString(e));
  return ESC_OK;
}

int esc_csv_check(const uint8_t* d_bytes, int64_t nbytes, const int64_t* d_field_end, const uint8_t* d_field_kind,
                  int64_t nsep, const int64_t* d_rec_end, int64_t nrows, int64_t first_field, int32_t ncols,
                  uint64_t* d_out, void* stream) {
  if (nbytes < 0 || nsep < 0 || nrows < 0 || ncols <= 0 || d_out == nullptr ||
      (nsep > 0 && (d_field_end == nullptr || d_field_kind == nullptr)) || (nrows > 0 && d_rec_end == nullptr))
    return fail(ESC_ERR_INVALID, "bad CSV check arguments");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  cudaError_t e = cudaMemsetAsync(d_out, 0xFF, 2 * sizeof(uint64_t), st);
  if (e != cudaSuccess) return fail(ESC_ERR_CUDA, std::string("CSV check init: ") + cudaGetErrorString(e));
  const int64_t work = nrows > nsep ? nrows : nsep;
  if (work == 0) return ESC_OK;
  esc::CsvCheck p;
  p.b = d_bytes;
  p.n = nbytes;
  p.field_end = reinterpret_cast<const long long*>(d_field_end);
  p.field_kind = d_field_kind;
  p.nsep = nsep;
  p.rec_end = reinterpret_cast<const long long*>(d_rec_end);
  p.nrows = nrows;
  p.first_field = first_field;
  p.ncols = ncols;
  p.out = reinterpret_cast<unsigned long long*>(d_out);
  const int sms = sm_count_cached();
  if (sms <= 0) return fail(ESC_ERR_CUDA, "no CUDA device");
  int64_t blocks = (work + 255) / 256;
  if (blocks > (int64_t)sms * 16) blocks = (int64_t)sms * 16;
  ++g_launches;
  esc::csv_check_kernel<<<(unsigned)blocks, 256, 0, st>>>(p);
  e = cudaGetLastError();
  if (e != cudaSuccess) return fail(ESC_ERR_CUDA, std::string("CSV check launch: ") + cudaGetErrorString(e));
  return ESC_OK;
}

}  // extern "C"
