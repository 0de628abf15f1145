// Where K5 and the interlevel prefix read a ray's packets from (composite.cu, interlevel.cu):
// the dense global slab [K][R] x 32 B (one process, or the dense exchange), or — after the
// sparse exchange — the received records themselves, through a [K][R] int32 index of record
// slots (-1: empty segment, identity packet) that vr_packets_index builds.  Both give the
// same packet values, so K5's fold is bit-identical either way; the index costs 4 B per
// (region, ray) instead of the dense slab's 32 B write + read.
#pragma once

#include "common.cuh"

namespace vr {

struct PacketSrc {
  const float4* pk;        // dense slab (index == nullptr)
  const float* extra;      // dense proposal-T slab [K][R] (dense mode, optional)
  const float* rec;        // records: [slots][width] {gidx, T, C0, C1, C2, A, D, L, order, (T')}
  const int32_t* index;    // [K][R] record slot or -1
  int width;
};

__device__ __forceinline__ PacketSrc dense_src(const float4* pk, const float* extra) {
  PacketSrc s;
  s.pk = pk;
  s.extra = extra;
  s.rec = nullptr;
  s.index = nullptr;
  s.width = 0;
  return s;
}

// order key of segment g = k * R + r (INT32_MAX: empty)
__device__ __forceinline__ int pk_key(const PacketSrc& s, int64_t g) {
  if (!s.index) return __float_as_int(s.pk[2 * g + 1].w);
  const int32_t i = __ldg(s.index + g);
  return i < 0 ? INT32_MAX : __float_as_int(__ldg(s.rec + (int64_t)i * s.width + 8));
}

// the packet's {T, C0, C1, C2} and {A, D, L, order} (a non-empty segment)
__device__ __forceinline__ void pk_load(const PacketSrc& s, int64_t g, float4& a, float4& b) {
  if (!s.index) {
    a = s.pk[2 * g];
    b = s.pk[2 * g + 1];
    return;
  }
  const float* r = s.rec + (int64_t)__ldg(s.index + g) * s.width;
  a = make_float4(r[1], r[2], r[3], r[4]);
  b = make_float4(r[5], r[6], r[7], r[8]);
}

// the proposal transmittance riding with the packet (interlevel; a non-empty segment)
__device__ __forceinline__ float pk_extra(const PacketSrc& s, int64_t g) {
  if (!s.index) return s.extra[g];
  return s.rec[(int64_t)__ldg(s.index + g) * s.width + 9];
}

}  // namespace vr
