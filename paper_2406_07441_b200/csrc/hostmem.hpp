// Host memory for the multi-GB setup arrays (a 40M-point cloud holds ~20 GB
// of CSR stencils, LS operators and packing temporaries).
//
// Two costs dominate setup at that size and neither is arithmetic: 4-KB page
// faults (the first touch of every page, serialised in the kernel when one
// thread zero-fills a whole vector) and zero-filling arrays that are about to
// be overwritten. BigAlloc maps large blocks directly with transparent huge
// pages requested (madvise(MADV_HUGEPAGE): 512x fewer faults) and leaves
// elements default-initialised on resize(), so the parallel loop that fills
// an array is also the one that first touches its pages.
#pragma once

#include <sys/mman.h>

#include <cstddef>
#include <cstdlib>
#include <new>
#include <utility>
#include <vector>

namespace kfb {

template <class T>
struct BigAlloc {
    using value_type = T;
    static constexpr size_t kMapBytes = size_t(4) << 20;  // mmap + THP from 4 MB up

    BigAlloc() noexcept = default;
    template <class U>
    BigAlloc(const BigAlloc<U>&) noexcept
    {
    }

    T* allocate(size_t n)
    {
        const size_t bytes = n * sizeof(T);
        if (bytes < kMapBytes) {
            void* p = std::malloc(bytes ? bytes : 1);
            if (!p) throw std::bad_alloc();
            return static_cast<T*>(p);
        }
        void* p = mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
        if (p == MAP_FAILED) throw std::bad_alloc();
        madvise(p, bytes, MADV_HUGEPAGE);
        return static_cast<T*>(p);
    }
    void deallocate(T* p, size_t n) noexcept
    {
        const size_t bytes = n * sizeof(T);
        if (bytes < kMapBytes)
            std::free(p);
        else
            munmap(p, bytes);
    }
    // resize() without a value leaves trivial elements uninitialised (the
    // filling loop touches them first); every other construction is normal
    template <class U, class... A>
    void construct(U* p, A&&... a)
    {
        if constexpr (sizeof...(A) == 0)
            ::new (static_cast<void*>(p)) U;
        else
            ::new (static_cast<void*>(p)) U(std::forward<A>(a)...);
    }
    template <class U>
    bool operator==(const BigAlloc<U>&) const noexcept
    {
        return true;
    }
    template <class U>
    bool operator!=(const BigAlloc<U>&) const noexcept
    {
        return false;
    }
};

template <class T>
using bvec = std::vector<T, BigAlloc<T>>;

// Parallel fill of a freshly resized array (first touch in parallel).
template <class V, class T>
void par_fill(V& v, const T& x)
{
    const long long n = static_cast<long long>(v.size());
    auto* d = v.data();
#pragma omp parallel for schedule(static)
    for (long long i = 0; i < n; ++i) d[i] = x;
}

// v = n copies of x, first touched by all threads.
template <class V, class T>
void fresh(V& v, size_t n, const T& x)
{
    v.clear();
    v.resize(n);
    par_fill(v, x);
}

}  // namespace kfb
