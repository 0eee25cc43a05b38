// egs_narrow.cpp — see egs_narrow.h.  The scalar loop (a compare and a
// truncating store per weight) runs at ~0.85 G weights/s per core on the GPU
// box's Xeon: 16 threads need ~28 ms for C4's 2 GB of int64 weights, longer
// than the 25.6 ms PCIe transfer it should hide behind.  The AVX-512 loop
// (vpminsq / vpmaxsq for the range, vpmovq{b,w,d} to narrow) reads at memory
// speed.
#include "egs_narrow.h"

#include <immintrin.h>

#include <algorithm>

namespace {

template <class W>
bool narrow_scalar(const int64_t* in, W* out, size_t count, int64_t wmax) {
  int64_t lo = 0, hi = 0;
  for (size_t i = 0; i < count; ++i) {
    const int64_t x = in[i];
    lo = std::min(lo, x);
    hi = std::max(hi, x);
    out[i] = static_cast<W>(x);
  }
  return lo < -wmax || hi > wmax;
}

// 8 weights per vector; the store width follows W.  Streaming (non-temporal)
// stores: the stage is read next by the DMA engine, not by this core, and
// they skip the line fill a plain store makes -- the upload is bound by
// host-memory traffic (DMA reads + these reads of the int64 weights).
// `out` is aligned to the store width (the caller's scalar head).
template <class W>
__attribute__((target("avx512f,avx512bw,avx512vl"))) inline void store8(W* out, __m512i v);
template <>
__attribute__((target("avx512f,avx512bw,avx512vl"))) inline void store8<int8_t>(int8_t* out,
                                                                               __m512i v) {
  _mm_stream_si64(reinterpret_cast<long long*>(out), _mm_cvtsi128_si64(_mm512_cvtepi64_epi8(v)));
}
template <>
__attribute__((target("avx512f,avx512bw,avx512vl"))) inline void store8<int16_t>(int16_t* out,
                                                                                __m512i v) {
  _mm_stream_si128(reinterpret_cast<__m128i*>(out), _mm512_cvtepi64_epi16(v));
}
template <>
__attribute__((target("avx512f,avx512bw,avx512vl"))) inline void store8<int32_t>(int32_t* out,
                                                                                __m512i v) {
  _mm256_stream_si256(reinterpret_cast<__m256i*>(out), _mm512_cvtepi64_epi32(v));
}

template <class W>
__attribute__((target("avx512f,avx512bw,avx512vl"))) bool narrow_avx512(const int64_t* in, W* out,
                                                                        size_t count,
                                                                        int64_t wmax) {
  __m512i lo0 = _mm512_setzero_si512(), hi0 = lo0, lo1 = lo0, hi1 = lo0;
  // scalar head up to the store width's alignment of out
  size_t i = 0;
  bool head_bad = false;
  while (i < count && (reinterpret_cast<uintptr_t>(out + i) & (8 * sizeof(W) - 1))) {
    head_bad |= narrow_scalar<W>(in + i, out + i, 1, wmax);
    ++i;
  }
  for (; i + 16 <= count; i += 16) {
    const __m512i a = _mm512_loadu_si512(in + i);
    const __m512i b = _mm512_loadu_si512(in + i + 8);
    lo0 = _mm512_min_epi64(lo0, a);
    hi0 = _mm512_max_epi64(hi0, a);
    lo1 = _mm512_min_epi64(lo1, b);
    hi1 = _mm512_max_epi64(hi1, b);
    store8<W>(out + i, a);
    store8<W>(out + i + 8, b);
  }
  _mm_sfence();
  const int64_t lo = _mm512_reduce_min_epi64(_mm512_min_epi64(lo0, lo1));
  const int64_t hi = _mm512_reduce_max_epi64(_mm512_max_epi64(hi0, hi1));
  const bool tail_bad = narrow_scalar<W>(in + i, out + i, count - i, wmax);
  return head_bad || tail_bad || lo < -wmax || hi > wmax;
}

void widen_scalar(const uint32_t* in, int64_t* out, size_t count) {
  for (size_t i = 0; i < count; ++i)
    out[i] = in[i] == 0xffffffffu ? INT64_MAX : static_cast<int64_t>(in[i]);
}

__attribute__((target("avx512f,avx512bw,avx512vl"))) void widen_avx512(const uint32_t* in,
                                                                      int64_t* out,
                                                                      size_t count) {
  const __m512i top32 = _mm512_set1_epi64(0xffffffffll), top64 = _mm512_set1_epi64(INT64_MAX);
  // scalar up to a 64-byte boundary of out, then streaming (non-temporal)
  // stores: the result is not re-read here, and they skip the line fills
  size_t i = 0;
  while (i < count && (reinterpret_cast<uintptr_t>(out + i) & 63u)) {
    widen_scalar(in + i, out + i, 1);
    ++i;
  }
  for (; i + 8 <= count; i += 8) {
    __m512i v = _mm512_cvtepu32_epi64(_mm256_loadu_si256(reinterpret_cast<const __m256i*>(in + i)));
    v = _mm512_mask_mov_epi64(v, _mm512_cmpeq_epi64_mask(v, top32), top64);
    _mm512_stream_si512(reinterpret_cast<__m512i*>(out + i), v);
  }
  _mm_sfence();
  widen_scalar(in + i, out + i, count - i);
}

bool have_avx512() {
  static const bool ok = __builtin_cpu_supports("avx512f") && __builtin_cpu_supports("avx512bw") &&
                         __builtin_cpu_supports("avx512vl");
  return ok;
}

template <class W>
bool narrow(const int64_t* in, W* out, size_t count, int64_t wmax) {
  return have_avx512() ? narrow_avx512<W>(in, out, count, wmax)
                       : narrow_scalar<W>(in, out, count, wmax);
}

}  // namespace

void egs_internal_widen_u32(const uint32_t* in, int64_t* out, size_t count) {
  if (have_avx512())
    widen_avx512(in, out, count);
  else
    widen_scalar(in, out, count);
}

bool egs_internal_narrow_i8(const int64_t* in, int8_t* out, size_t count, int64_t wmax) {
  return narrow<int8_t>(in, out, count, wmax);
}
bool egs_internal_narrow_i16(const int64_t* in, int16_t* out, size_t count, int64_t wmax) {
  return narrow<int16_t>(in, out, count, wmax);
}
bool egs_internal_narrow_i32(const int64_t* in, int32_t* out, size_t count, int64_t wmax) {
  return narrow<int32_t>(in, out, count, wmax);
}
