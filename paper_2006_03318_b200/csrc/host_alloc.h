// host_alloc.h -- host allocator for multi-GB host-side arrays (graph
// compiler, trace reader).
#pragma once
#include <vector>
// Large arrays: 2 MB-aligned blocks
// advised as transparent huge pages (the boxes run THP in madvise mode), so
// first-touch of multi-GB compile state costs 512x fewer page faults.
#include <sys/mman.h>
#include <cstdlib>
#include <new>
template <class T>
struct HugeAlloc {
  using value_type = T;
  HugeAlloc() = default;
  template <class U>
  HugeAlloc(const HugeAlloc<U>&) {}
  T* allocate(std::size_t n) {
    const std::size_t bytes = n * sizeof(T);
    if (bytes < (4u << 20)) {
      void* p = std::malloc(bytes ? bytes : 1);
      if (!p) throw std::bad_alloc();
      return static_cast<T*>(p);
    }
    const std::size_t al = std::size_t(2) << 20;
    void* p = std::aligned_alloc(al, (bytes + al - 1) / al * al);
    if (!p) throw std::bad_alloc();
    madvise(p, bytes, MADV_HUGEPAGE);
    return static_cast<T*>(p);
  }
  void deallocate(T* p, std::size_t) { std::free(p); }
  template <class U>
  bool operator==(const HugeAlloc<U>&) const { return true; }
  template <class U>
  bool operator!=(const HugeAlloc<U>&) const { return false; }
};
template <class T>
using hvec = std::vector<T, HugeAlloc<T>>;
