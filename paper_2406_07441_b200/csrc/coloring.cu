// Sweep-ordering variants on the device.
//
// The reference colours the cloud with a sequential greedy pass
// (color_points, coloring.cpp:23-52): colours depend on the point numbering,
// and a loaded cloud with no locality needs many more colours than an O-grid
// (a shuffled 640,000-point O-grid: 8 instead of 4, profiles/r01_orderings.txt),
// each one a dependent launch pair of the LU-SGS sweeps. Two stated variants
// of the sweep ORDER are built here; each changes which neighbours count as
// "lower" / "upper" in forward_sweep / backward_sweep (implicit.cpp:164-165),
// so they are validated against the reference run with the same plan (the
// reference accepts any SweepPlan, driver.hpp:104-106) and, at solution level,
// against the reference's own ordering (tests/test_gpu_orderings.py):
//
//  * jones_plassmann: a parallel colouring of the symmetrised graph
//    (symmetrized_connectivity, coloring.cpp:7-21). Every round, each
//    uncoloured point whose priority beats all its uncoloured neighbours takes
//    the smallest colour none of its neighbours holds; the round's winners are
//    independent, so the two phases (elect, colour) are race-free and the
//    result is deterministic. Priorities: a hash of the point id ("random"),
//    or the degree first ("largest degree first"), hash as the tie-break.
//    Iterated-greedy passes (Culberson) then recolour class by class, each
//    class in parallel, while they remove colours. Quality on an O-grid
//    (king's-graph stencils): 7 colours, like the reference's own greedy
//    over a Morton or random numbering (7 / 8); only the generator's natural
//    ring-by-ring numbering gives greedy its 4.
//  * wall_first_levels: the paper's Algorithm 5: wall,
//    interior and outer points are swept as separate groups, each in its own
//    colour order -- a level = (kind, colour), levels ordered wall < interior
//    < outer, empty levels dropped.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <string>
#include <vector>

#include "cloud.hpp"
#include "solver.hpp"

namespace kfb {

namespace {

void ckc(cudaError_t e, const char* what)
{
    if (e != cudaSuccess)
        throw SolverError(KF_CUDA, std::string("colouring: ") + what + ": " + cudaGetErrorString(e));
}

__host__ __device__ inline uint32_t mix32(uint32_t x, uint32_t seed)
{
    // murmur3 finaliser of (id ^ seed)
    x ^= seed * 0x9e3779b9u;
    x ^= x >> 16;
    x *= 0x85ebca6bu;
    x ^= x >> 13;
    x *= 0xc2b2ae35u;
    x ^= x >> 16;
    return x;
}

// priority: higher wins; ties by the smaller id
__global__ void k_jp_priority(int n, const long long* off, int mode, uint32_t seed, unsigned long long* prio)
{
    const int v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= n) return;
    const unsigned long long h = mix32(static_cast<uint32_t>(v), seed);
    const unsigned long long deg = static_cast<unsigned long long>(off[v + 1] - off[v]);
    prio[v] = mode == 1 ? (deg << 32) | h : h;
}

__device__ __forceinline__ bool beats(unsigned long long pa, int a, unsigned long long pb, int b)
{
    return pa > pb || (pa == pb && a < b);
}

// phase 1: an uncoloured point whose priority beats every uncoloured
// neighbour is elected (colours are read-only in this phase)
__global__ void k_jp_elect(int n, const long long* off, const int* adj, const unsigned long long* prio,
                           const int* color, unsigned char* win, int* remaining)
{
    const int v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= n) return;
    win[v] = 0;
    if (color[v] != 0) return;
    // one atomic per warp: the still-uncoloured lanes are the active ones
    const unsigned act = __activemask();
    if ((threadIdx.x & 31) == __ffs(act) - 1) atomicAdd(remaining, __popc(act));
    const unsigned long long pv = prio[v];
    for (long long k = off[v]; k < off[v + 1]; ++k) {
        const int q = adj[k];
        if (color[q] == 0 && !beats(pv, v, prio[q], q)) return;
    }
    win[v] = 1;
}

// phase 2: the winners (an independent set) take the smallest colour that no
// neighbour holds
__global__ void k_jp_color(int n, const long long* off, const int* adj, const unsigned char* win, int* color)
{
    const int v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= n || !win[v]) return;
    unsigned long long used = 0;  // colours 1..64 held by neighbours
    for (long long k = off[v]; k < off[v + 1]; ++k) {
        const int c = color[adj[k]];
        if (c >= 1 && c <= 64) used |= 1ull << (c - 1);
    }
    int pick = __ffsll(static_cast<long long>(~used));  // lowest free colour <= 64, 0 if none
    if (pick == 0) {
        // a hub with all of 1..64 around it: search upwards (colours > 64
        // never conflict with a pick <= 64, so only this case needs it)
        for (int c = 65;; ++c) {
            bool taken = false;
            for (long long k = off[v]; k < off[v + 1] && !taken; ++k) taken = color[adj[k]] == c;
            if (!taken) {
                pick = c;
                break;
            }
        }
    }
    color[v] = pick;
}

// Iterated greedy (Culberson): a pass recolours the classes of the current
// colouring one after another, each class at once (a class is an independent
// set, so its points never see each other), first-fit against the NEW colours
// of the classes already passed. The count never increases; the pass order
// is the classes in descending order.
__global__ void k_ig_class(int n, const long long* off, const int* adj, const int* old, int k, int* nw)
{
    const int v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= n || old[v] != k) return;
    unsigned long long used = 0;
    for (long long e = off[v]; e < off[v + 1]; ++e) {
        const int c = nw[adj[e]];
        if (c >= 1 && c <= 64) used |= 1ull << (c - 1);
    }
    int pick = __ffsll(static_cast<long long>(~used));
    if (pick == 0) {
        for (int c = 65;; ++c) {
            bool taken = false;
            for (long long e = off[v]; e < off[v + 1] && !taken; ++e) taken = nw[adj[e]] == c;
            if (!taken) {
                pick = c;
                break;
            }
        }
    }
    nw[v] = pick;
}

}  // namespace

// Symmetrised adjacency (symmetrized_connectivity, coloring.cpp:7-21): sorted,
// duplicates and self entries dropped, 64-bit offsets.
static void symmetrised(const Cloud& c, std::vector<long long>& aoff, std::vector<int>& adj)
{
    const int n = c.n;
    std::vector<long long> cnt(n + 1, 0);
    for (int i = 0; i < n; ++i)
        for (int k = c.nbr.off[i]; k < c.nbr.off[i + 1]; ++k) {
            ++cnt[i + 1];
            ++cnt[c.nbr.idx[k] + 1];
        }
    for (int i = 0; i < n; ++i) cnt[i + 1] += cnt[i];
    std::vector<int> raw(cnt[n]);
    std::vector<long long> pos(cnt.begin(), cnt.end() - 1);
    for (int i = 0; i < n; ++i)
        for (int k = c.nbr.off[i]; k < c.nbr.off[i + 1]; ++k) {
            const int q = c.nbr.idx[k];
            raw[pos[i]++] = q;
            raw[pos[q]++] = i;
        }
    std::vector<int> len(n);
#pragma omp parallel for schedule(static)
    for (int i = 0; i < n; ++i) {
        int* a = raw.data() + cnt[i];
        int* e = raw.data() + cnt[i + 1];
        std::sort(a, e);
        e = std::unique(a, e);
        e = std::remove(a, e, i);
        len[i] = static_cast<int>(e - a);
    }
    aoff.assign(n + 1, 0);
    for (int i = 0; i < n; ++i) aoff[i + 1] = aoff[i] + len[i];
    adj.resize(aoff[n]);
#pragma omp parallel for schedule(static)
    for (int i = 0; i < n; ++i) std::copy(raw.data() + cnt[i], raw.data() + cnt[i] + len[i], adj.data() + aoff[i]);
}

int jones_plassmann_colors(Cloud& c, int device, int mode, unsigned seed, int* rounds_out)
{
    const int n = c.n;
    if (n == 0) {
        c.color.clear();
        c.n_colors = 0;
        return 0;
    }
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
        throw SolverError(KF_CUDA, "no CUDA device available (the B200 path has no CPU fallback)");
    ckc(cudaSetDevice(device), "cudaSetDevice");
    std::vector<long long> aoff;
    std::vector<int> adj;
    symmetrised(c, aoff, adj);
    cudaStream_t s;
    ckc(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "stream");
    long long* d_off = nullptr;
    int* d_adj = nullptr;
    int* d_color = nullptr;
    int* d_rem = nullptr;
    unsigned long long* d_prio = nullptr;
    unsigned char* d_win = nullptr;
    int* d_new = nullptr;
    auto freeall = [&] {
        cudaFree(d_new);
        cudaFree(d_off);
        cudaFree(d_adj);
        cudaFree(d_color);
        cudaFree(d_rem);
        cudaFree(d_prio);
        cudaFree(d_win);
        cudaStreamDestroy(s);
    };
    try {
        ckc(cudaMalloc(&d_off, sizeof(long long) * (n + 1)), "malloc");
        ckc(cudaMalloc(&d_adj, sizeof(int) * std::max<size_t>(adj.size(), 1)), "malloc");
        ckc(cudaMalloc(&d_color, sizeof(int) * n), "malloc");
        ckc(cudaMalloc(&d_rem, sizeof(int) * 64), "malloc");
        ckc(cudaMalloc(&d_prio, sizeof(unsigned long long) * n), "malloc");
        ckc(cudaMalloc(&d_win, n), "malloc");
        ckc(cudaMemcpyAsync(d_off, aoff.data(), sizeof(long long) * (n + 1), cudaMemcpyHostToDevice, s), "H2D");
        if (!adj.empty())
            ckc(cudaMemcpyAsync(d_adj, adj.data(), sizeof(int) * adj.size(), cudaMemcpyHostToDevice, s), "H2D");
        ckc(cudaMemsetAsync(d_color, 0, sizeof(int) * n, s), "memset");
        ckc(cudaMemsetAsync(d_rem, 0, sizeof(int) * 64, s), "memset");
        const int T = 256, B = (n + T - 1) / T;
        k_jp_priority<<<B, T, 0, s>>>(n, d_off, mode, seed, d_prio);
        // rounds in batches of 8 (one remaining-counter per round) between
        // host checks
        int rounds = 0;
        std::vector<int> rem(8);
        for (;;) {
            for (int r = 0; r < 8; ++r) {
                k_jp_elect<<<B, T, 0, s>>>(n, d_off, d_adj, d_prio, d_color, d_win, d_rem + r);
                k_jp_color<<<B, T, 0, s>>>(n, d_off, d_adj, d_win, d_color);
            }
            ckc(cudaGetLastError(), "launch");
            ckc(cudaMemcpyAsync(rem.data(), d_rem, sizeof(int) * 8, cudaMemcpyDeviceToHost, s), "D2H");
            ckc(cudaMemsetAsync(d_rem, 0, sizeof(int) * 8, s), "memset");
            ckc(cudaStreamSynchronize(s), "sync");
            int done_at = -1;
            for (int r = 0; r < 8; ++r)
                if (rem[r] == 0) {
                    done_at = r;
                    break;
                }
            if (done_at >= 0) {
                rounds += done_at;
                break;
            }
            rounds += 8;
            if (rounds > 4 * n + 64) throw SolverError(KF_RUNTIME, "colouring: no progress");
        }
        // iterated-greedy passes while they still remove a colour (at most 4)
        int nc = 0;
        {
            std::vector<int> h(n);
            ckc(cudaMemcpyAsync(h.data(), d_color, sizeof(int) * n, cudaMemcpyDeviceToHost, s), "D2H");
            ckc(cudaStreamSynchronize(s), "sync");
            nc = *std::max_element(h.begin(), h.end());
        }
        ckc(cudaMalloc(&d_new, sizeof(int) * n), "malloc");
        for (int pass = 0; pass < 4; ++pass) {
            ckc(cudaMemsetAsync(d_new, 0, sizeof(int) * n, s), "memset");
            for (int k = nc; k >= 1; --k) k_ig_class<<<B, T, 0, s>>>(n, d_off, d_adj, d_color, k, d_new);
            ckc(cudaGetLastError(), "launch");
            std::swap(d_color, d_new);
            std::vector<int> h(n);
            ckc(cudaMemcpyAsync(h.data(), d_color, sizeof(int) * n, cudaMemcpyDeviceToHost, s), "D2H");
            ckc(cudaStreamSynchronize(s), "sync");
            const int m = *std::max_element(h.begin(), h.end());
            if (m >= nc) {
                nc = m;
                break;
            }
            nc = m;
        }
        c.color.assign(n, 0);
        ckc(cudaMemcpyAsync(c.color.data(), d_color, sizeof(int) * n, cudaMemcpyDeviceToHost, s), "D2H");
        ckc(cudaStreamSynchronize(s), "sync");
        if (rounds_out) *rounds_out = rounds;
    } catch (...) {
        freeall();
        throw;
    }
    freeall();
    c.n_colors = *std::max_element(c.color.begin(), c.color.end());
    return c.n_colors;
}

int wall_first_levels(Cloud& c)
{
    const int n = c.n;
    const int C = std::max(c.n_colors, 1);
    // level (kind rank, colour): wall 0, interior 1, outer 2 (Algorithm 5 order)
    std::vector<int> used(3 * C + 1, 0);
    auto level = [&](int p) {
        const int k = c.kind[p] == kWall ? 0 : c.kind[p] == kInterior ? 1 : 2;
        return k * C + c.color[p];
    };
    for (int p = 0; p < n; ++p) used[level(p)] = 1;
    std::vector<int> map(3 * C + 1, 0);
    int m = 0;
    for (int l = 1; l <= 3 * C; ++l)
        if (used[l]) map[l] = ++m;
    bvec<int> nc(n);
    for (int p = 0; p < n; ++p) nc[p] = map[level(p)];
    c.color.swap(nc);
    c.n_colors = m;
    return m;
}

}  // namespace kfb
