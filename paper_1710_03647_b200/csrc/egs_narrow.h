// egs_narrow.h — host-side narrowing of the reference's int64 edge weights
// (arena.hpp:13) to the upload width (int8 / int16 / int32), range-checked
// against |w| <= wmax.  Internal to libegs_b200.so (egs_solver.cu's
// upload_weights); AVX-512 when the host has it, scalar otherwise.
#pragma once

#include <cstddef>
#include <cstdint>

// out[i] = (W)in[i] for i < count; returns true if some |in[i]| > wmax
bool egs_internal_narrow_i8(const int64_t* in, int8_t* out, size_t count, int64_t wmax);
bool egs_internal_narrow_i16(const int64_t* in, int16_t* out, size_t count, int64_t wmax);
bool egs_internal_narrow_i32(const int64_t* in, int32_t* out, size_t count, int64_t wmax);

// The other way, for the measure read back as 32-bit device values: out[i] =
// in[i], except the device top (all ones) -> INT64_MAX (energy.hpp:16).
void egs_internal_widen_u32(const uint32_t* in, int64_t* out, size_t count);
