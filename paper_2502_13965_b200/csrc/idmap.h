// Host-side id map of the autx C ABI (autx_api.cu): active call id -> call-table row.
#pragma once
#include <algorithm>
#include <cstddef>
#include <cstdint>
#include <climits>
#include <vector>

// Active call id -> call-table row: open addressing with linear probing over flat arrays (the
// per-step path looks up, inserts and erases one entry per completion / arrival; no node
// allocation per insert as with std::unordered_map, and compaction remaps by one array sweep).
class IdMap {
  std::vector<uint64_t> key_;
  std::vector<uint32_t> val_;
  std::vector<uint8_t> st_;  // 0 empty, 1 full, 2 erased
  size_t mask_ = 0, n_ = 0, used_ = 0;  // used_ = full + erased
  static uint64_t mix(uint64_t x) {
    x ^= x >> 30; x *= 0xbf58476d1ce4e5b9ull; x ^= x >> 27; x *= 0x94d049bb133111ebull; return x ^ (x >> 31);
  }
  void rebuild(size_t cap) {
    std::vector<uint64_t> k(cap);
    std::vector<uint32_t> v(cap);
    std::vector<uint8_t> st(cap, 0);
    for (size_t i = 0; i < st_.size(); ++i)
      if (st_[i] == 1) {
        size_t j = mix(key_[i]) & (cap - 1);
        while (st[j]) j = (j + 1) & (cap - 1);
        k[j] = key_[i]; v[j] = val_[i]; st[j] = 1;
      }
    key_.swap(k); val_.swap(v); st_.swap(st);
    mask_ = cap - 1;
    used_ = n_;
  }
  size_t slot_of(uint64_t k) const {  // index of k, or SIZE_MAX
    if (st_.empty()) return SIZE_MAX;
    for (size_t j = mix(k) & mask_;; j = (j + 1) & mask_) {
      if (st_[j] == 0) return SIZE_MAX;
      if (st_[j] == 1 && key_[j] == k) return j;
    }
  }
 public:
  void reserve(size_t n) {
    size_t cap = 16;
    while (cap < 2 * n) cap <<= 1;
    if (cap > st_.size()) rebuild(cap);
  }
  size_t size() const { return n_; }
  bool empty() const { return n_ == 0; }
  uint32_t* find(uint64_t k) {
    const size_t j = slot_of(k);
    return j == SIZE_MAX ? nullptr : &val_[j];
  }
  size_t count(uint64_t k) const { return slot_of(k) == SIZE_MAX ? 0 : 1; }
  void erase(uint64_t k) {
    const size_t j = slot_of(k);
    if (j != SIZE_MAX) { st_[j] = 2; --n_; }
  }
  uint32_t& operator[](uint64_t k) {
    if (uint32_t* v = find(k)) return *v;
    if (4 * (used_ + 1) > 3 * st_.size()) rebuild(std::max<size_t>(16, 2 * (n_ + 1) > st_.size() / 2 ? 2 * st_.size() : st_.size()));
    size_t j = mix(k) & mask_;
    while (st_[j] == 1) j = (j + 1) & mask_;
    if (st_[j] == 0) ++used_;
    st_[j] = 1; key_[j] = k; val_[j] = 0; ++n_;
    return val_[j];
  }
  template <class F> void for_each(F f) {
    for (size_t i = 0; i < st_.size(); ++i)
      if (st_[i] == 1) f(key_[i], val_[i]);
  }
};

