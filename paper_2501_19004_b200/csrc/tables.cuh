// Open-addressing community tables over shared or global memory (the device
// counterpart of the reference's slab tables, compact_hashtable.hpp:28-122):
// power-of-two capacity, multiplicative hash, empty key 0xFFFFFFFF, and the
// reference's four probing modes (lvn_params.probing, probe_advance in
// compact_hashtable.hpp:60-82): linear, quadratic (doubling strides), double
// hashing (stride key mod p2, forced odd so it cycles a power-of-two table)
// and quadratic-double (stride = 2 stride + key mod p2); as in the reference
// the walk turns linear after 2x capacity probes, so a free or matching slot
// is always reached. Capacity is always >= 2x the distinct keys that can arrive,
// so probing terminates. insert() returns the slot it claimed for a new key
// (-1 when the key was already present), so callers can keep a list of live
// slots: scans then touch only live entries and clearing touches only them.
#pragma once

#include "common.cuh"

namespace lvn {

// probing mode of the tables of this translation unit (set_probing_*; 0
// linear, 1 quadratic, 2 double hashing, 3 quadratic-double)
static __constant__ int c_probing;

// one probe step of the walk: slot h, attempt number, stride state
__device__ __forceinline__ u32 probe_next(u32 h, u32 mask, u32 attempt, u32& stride, u32 kmod) {
  const int mode = c_probing;
  if (mode == 0 || attempt + 1 >= 2 * (mask + 1)) return (h + 1) & mask;
  if (mode == 1) {
    const u32 n = (h + stride) & mask;
    stride *= 2;
    return n;
  }
  if (mode == 2) return (h + (kmod | 1u)) & mask;
  const u32 n = (h + stride) & mask;
  stride = 2 * stride + kmod;
  return n;
}
__device__ __forceinline__ u32 probe_kmod(u32 key, u32 log_size) {
  return key % ((2u << log_size) + 1u);  // p2 = 2 x capacity + 1
}

__device__ __forceinline__ u32 table_log(u64 deg, u32 min_log) {
  const u32 l = ceil_log2_u64(2 * deg);
  return l > min_log ? l : min_log;
}

// ---- table flavours ---------------------------------------------------------
struct PackedF32 {  // value_bits == 32: one 64-bit slot (key << 32 | float bits), one CAS per update
  using V = float;
  static constexpr size_t kSlotBytes = 8;
  ull* s;
  __device__ PackedF32(void* base, u64 slots) : s(static_cast<ull*>(base)) { (void)slots; }
  __device__ __forceinline__ void clear(u32 i) const { s[i] = kEmptySlot64; }
  // first probe inline; a collision continues out of line (keeps the probe
  // state out of the callers' registers)
  __device__ __forceinline__ int insert(u32 log_size, u32 key, float w) const {
    const u32 h = slot_hash(key, log_size);
    const ull cur = reinterpret_cast<volatile ull*>(s)[h];
    const u32 k = u32(cur >> 32);
    if (k == key || k == kEmpty) {
      const ull want = (ull(key) << 32) | __float_as_uint(__uint_as_float(u32(cur)) + w);
      if (atomicCAS(&s[h], cur, want) == cur) return k == kEmpty ? int(h) : -1;
      return insert_from(log_size, key, w, h, 0u);  // lost a race: retry the same slot
    }
    return insert_from(log_size, key, w, h, 1u);
  }
  __device__ __noinline__ int insert_from(u32 log_size, u32 key, float w, u32 h, u32 advance) const {
    const u32 mask = (1u << log_size) - 1u;
    u32 attempt = 0, stride = 1;
    const u32 kmod = c_probing ? probe_kmod(key, log_size) : 0u;
    if (advance) h = probe_next(h, mask, attempt++, stride, kmod);
    while (true) {
      const ull cur = reinterpret_cast<volatile ull*>(s)[h];
      const u32 k = u32(cur >> 32);
      if (k == key || k == kEmpty) {
        const float nv = __uint_as_float(u32(cur)) + w;
        const ull want = (ull(key) << 32) | __float_as_uint(nv);
        if (atomicCAS(&s[h], cur, want) == cur) return k == kEmpty ? int(h) : -1;
      } else {
        h = probe_next(h, mask, attempt++, stride, kmod);
      }
    }
  }
  __device__ __forceinline__ bool read(u32 i, u32& key, double& val) const {
    const ull x = s[i];
    key = u32(x >> 32);
    val = double(__uint_as_float(u32(x)));
    return key != kEmpty;
  }
};

struct SplitF64 {  // value_bits == 64: u32 key array + fp64 value array
  using V = double;
  static constexpr size_t kSlotBytes = 12;
  u32* k;
  double* v;
  __device__ SplitF64(void* base, u64 slots)
      : k(reinterpret_cast<u32*>(static_cast<double*>(base) + slots)),
        v(static_cast<double*>(base)) {}
  __device__ __forceinline__ void clear(u32 i) const {
    k[i] = kEmpty;
    v[i] = 0.0;
  }
  __device__ __forceinline__ int insert(u32 log_size, u32 key, double w) const {
    const u32 h = slot_hash(key, log_size);
    u32 cur = reinterpret_cast<volatile u32*>(k)[h];
    int claimed = -1;
    if (cur == kEmpty) {
      cur = atomicCAS(&k[h], kEmpty, key);
      if (cur == kEmpty) cur = key, claimed = int(h);
    }
    if (cur == key) {
      atomicAdd(&v[h], w);
      return claimed;
    }
    return insert_from(log_size, key, w, h);
  }
  __device__ __noinline__ int insert_from(u32 log_size, u32 key, double w, u32 h) const {
    const u32 mask = (1u << log_size) - 1u;
    u32 attempt = 0, stride = 1;
    const u32 kmod = c_probing ? probe_kmod(key, log_size) : 0u;
    h = probe_next(h, mask, attempt++, stride, kmod);
    while (true) {
      u32 cur = reinterpret_cast<volatile u32*>(k)[h];
      int claimed = -1;
      if (cur == kEmpty) {
        cur = atomicCAS(&k[h], kEmpty, key);
        if (cur == kEmpty) cur = key, claimed = int(h);
      }
      if (cur == key) {
        atomicAdd(&v[h], w);
        return claimed;
      }
      h = probe_next(h, mask, attempt++, stride, kmod);
    }
  }
  __device__ __forceinline__ bool read(u32 i, u32& key, double& val) const {
    key = k[i];
    val = v[i];
    return key != kEmpty;
  }
};

}  // namespace lvn
