// vate_registry.cuh -- device-side insert into the host registry.
//
// SlidingHostSet.update (pipeline.py:50-52) sets last[aip] = t for every
// distinct aip of a slice.  On the device every packet probes the table; all
// writers of one call store the same t, so plain stores are race-free.  Keys
// are u64 (the reference keeps arbitrary Python ints, estimator.py:67-81).
#pragma once

#include "vate_internal.cuh"

namespace vate {

constexpr uint64_t kRegSalt = 0x2545F4914F6CDD1Dull;
constexpr int kMaxProbe = 64;

// Home slot of a key: linear probing starts at an EVEN slot, so the first two
// probes share one 32-byte sector and one 256-bit load (ld_pair) answers both
// -- at load factor <= 0.6 most lookups end inside that first sector.
__device__ __forceinline__ uint64_t reg_home(uint64_t key, uint64_t mask) {
  return (mix64(key ^ kRegSalt) & mask) & ~1ull;
}

// Slots s and s+1 (s even: one aligned 32-byte sector) in one load.
__device__ __forceinline__ void ld_pair(const RegEntry* p, RegEntry& a, RegEntry& b,
                                        bool keep = false) {
  unsigned long long k0, l0, k1, l1;
  if (keep)
    asm volatile("ld.global.L2::cache_hint.v4.u64 {%0,%1,%2,%3}, [%4], %5;"
                 : "=l"(k0), "=l"(l0), "=l"(k1), "=l"(l1)
                 : "l"(p), "l"(l2_keep_policy()));
  else
    asm volatile("ld.global.v4.u64 {%0,%1,%2,%3}, [%4];"
                 : "=l"(k0), "=l"(l0), "=l"(k1), "=l"(l1)
                 : "l"(p));
  a.key = k0;
  a.last = (long long)l0;
  b.key = k1;
  b.last = (long long)l1;
}

// The scan's stamp of a found key (its loaded `last` differed from t).
__device__ __forceinline__ void reg_stamp(const RegRef& R, uint64_t slot, long long t) {
  if (R.stamp_max && R.l2_keep)
    asm volatile("red.relaxed.gpu.global.max.L2::cache_hint.s64 [%0], %1, %2;"
                 ::"l"(&R.table[slot].last), "l"(t), "l"(l2_keep_policy()) : "memory");
  else if (R.stamp_max)
    asm volatile("red.relaxed.gpu.global.max.s64 [%0], %1;" ::"l"(&R.table[slot].last), "l"(t)
                 : "memory");
  else
    R.table[slot].last = t;
}

__device__ __forceinline__ void reg_touch(RegEntry* e, long long t, bool use_max) {
  if (use_max) {
    atomicMax(&e->last, t);
  } else if (*((volatile long long*)&e->last) != t) {
    e->last = t;
  }
}

// Claim or find `key` at slot e (seen empty by a weak load): the CAS settles
// races; returns true when the key is (now) stored there.
__device__ __forceinline__ bool reg_claim(const RegRef& R, RegEntry* e, uint64_t key, long long t,
                                          bool use_max) {
  const unsigned long long prev = atomicCAS(&e->key, kEmptyKey, key);
  if (prev == kEmptyKey) {
    atomicAdd(R.count, 1ull);
    reg_touch(e, t, use_max);
    return true;
  }
  if (prev == key) {
    reg_touch(e, t, use_max);
    return true;
  }
  return false;  // another key took the slot first
}

// Insert-or-touch, one 32-byte sector (two slots, one 256-bit load) per probe
// step.  Weak loads are safe here: a slot's key changes only once (empty ->
// key) within a launch and there are no deletions, so a stale "empty" only
// sends us to the CAS, which reports the truth.  use_max is only used when
// draining the overflow list, where entries of several calls meet (identical
// to overwrite whenever slice indices are non-decreasing, as Pipeline.run
// feeds them).
//
// skip_home: the caller's own load saw the home sector full of other keys, so
// the walk starts at the next sector (non-empty keys never change).  Without
// use_max a found key is stamped from the loaded `last` (a stale read only
// repeats a store of the same t), with no second dependent load.
__device__ __forceinline__ void reg_insert(const RegRef& R, uint64_t key, long long t,
                                           bool use_max, bool skip_home = false) {
  if (key == kEmptyKey) {  // the one key that collides with the empty marker
    RegEntry* e = R.table + (R.mask + 1);
    if (atomicExch(R.special, 1u) == 0u) atomicAdd(R.count, 1ull);
    reg_touch(e, t, use_max);
    return;
  }
  uint64_t h = reg_home(key, R.mask);
  if (skip_home) h = (h + 2) & R.mask;
#pragma unroll 1
  for (int step = skip_home ? 1 : 0; step < kMaxProbe / 2; ++step) {
    RegEntry a, b;
    ld_pair(R.table + h, a, b, R.l2_keep);
    if (a.key == key) {
      if (use_max) reg_touch(R.table + h, t, true);
      else if (a.last != t) reg_stamp(R, h, t);
      return;
    }
    if (a.key == kEmptyKey && reg_claim(R, R.table + h, key, t, use_max)) return;
    // slot h is (now) some other key: b is next in the probe sequence
    if (b.key == key) {
      if (use_max) reg_touch(R.table + h + 1, t, true);
      else if (b.last != t) reg_stamp(R, h + 1, t);
      return;
    }
    if (b.key == kEmptyKey && reg_claim(R, R.table + h + 1, key, t, use_max)) return;
    h = (h + 2) & R.mask;  // both slots hold other keys (non-empty keys never change)
  }
  // probe limit: park it; the host drains (grows + reinserts) before any read
  unsigned long long slot = atomicAdd(R.ovf_n, 1ull);
  if (slot < R.ovf_cap) {
    R.ovf[slot].key = key;
    R.ovf[slot].last = t;
  }
}

}  // namespace vate
