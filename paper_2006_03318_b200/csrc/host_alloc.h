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

// Same allocator without value-initialisation: `uvec<T> v(n)` leaves POD
// elements unwritten (for arrays a builder overwrites completely, so the
// first touch happens on the writer threads instead of in a serial zero fill).
template <class T>
struct NoInitAlloc : HugeAlloc<T> {
  using value_type = T;
  template <class U>
  struct rebind { using other = NoInitAlloc<U>; };
  NoInitAlloc() = default;
  template <class U>
  NoInitAlloc(const NoInitAlloc<U>&) {}
  template <class U, class... A>
  void construct(U* p, A&&... a) {
    if constexpr (sizeof...(A) == 0)
      ::new (static_cast<void*>(p)) U;
    else
      ::new (static_cast<void*>(p)) U(static_cast<A&&>(a)...);
  }
};
template <class T>
using uvec = std::vector<T, NoInitAlloc<T>>;
