// Host-side ingestion. See cloud.hpp. Formulas follow the reference in
// evaluation order (compiled with -ffp-contract=off, no -march) so that the
// generated geometry, split stencils, LS weights and colours are bitwise the
// reference's; only the storage (flat CSR) differs.
#include "cloud.hpp"

#include <chrono>
#include <cstdio>
#include <cstdlib>

#include <algorithm>
#include <cctype>
#include <cerrno>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <exception>
#include <limits>
#include <thread>

#include <omp.h>

namespace kfb {

namespace {

constexpr double kSingularDetEps = 1e-12;  // pointcloud.hpp:50

struct Naca4 {
    double m, p, t;
};

// parse_naca, pointcloud.cpp:21-41
Naca4 parse_digits(const std::string& d)
{
    bool ok = d.size() == 4;
    for (char ch : d) ok = ok && std::isdigit(static_cast<unsigned char>(ch));
    if (!ok)
        throw IngestError(1, "invalid NACA code '" + d + "' (expected 4 digits)");
    Naca4 s;
    s.m = (d[0] - '0') / 100.0;
    s.p = (d[1] - '0') / 10.0;
    s.t = ((d[2] - '0') * 10 + (d[3] - '0')) / 100.0;
    if (s.t <= 0.0) throw IngestError(1, "invalid NACA code '" + d + "' (zero thickness)");
    if (s.m > 0.0 && s.p == 0.0)
        throw IngestError(1, "invalid NACA code '" + d + "' (camber without camber position)");
    return s;
}

// Closed-TE thickness polynomial and its slope, pointcloud.cpp:43-55
double half_thickness(const Naca4& s, double x)
{
    return 5.0 * s.t *
           (0.2969 * std::sqrt(x) - 0.1260 * x - 0.3516 * x * x + 0.2843 * x * x * x -
            0.1036 * x * x * x * x);
}
double half_thickness_dx(const Naca4& s, double x)
{
    return 5.0 * s.t *
           (0.14845 / std::sqrt(x) - 0.1260 - 0.7032 * x + 0.8529 * x * x -
            0.4144 * x * x * x);
}

// Mean camber line, slope, curvature, pointcloud.cpp:57-76
double camber_y(const Naca4& s, double x)
{
    if (s.m == 0.0) return 0.0;
    if (x < s.p) return s.m / (s.p * s.p) * (2.0 * s.p * x - x * x);
    return s.m / ((1.0 - s.p) * (1.0 - s.p)) * ((1.0 - 2.0 * s.p) + 2.0 * s.p * x - x * x);
}
double camber_dx(const Naca4& s, double x)
{
    if (s.m == 0.0) return 0.0;
    if (x < s.p) return 2.0 * s.m / (s.p * s.p) * (s.p - x);
    return 2.0 * s.m / ((1.0 - s.p) * (1.0 - s.p)) * (s.p - x);
}
double camber_dxx(const Naca4& s, double x)
{
    if (s.m == 0.0) return 0.0;
    if (x < s.p) return -2.0 * s.m / (s.p * s.p);
    return -2.0 * s.m / ((1.0 - s.p) * (1.0 - s.p));
}

struct WallSample {
    double x, y, nx, ny;
};

// Surface point + outward normal at polar parameter theta, pointcloud.cpp:83-135
WallSample surface_at(const Naca4& s, double theta)
{
    WallSample o;
    const double xc = 0.5 * (1.0 + std::cos(theta));
    const bool upper = theta < M_PI;
    const double side = upper ? 1.0 : -1.0;
    if (theta == 0.0) {
        const double slope = camber_dx(s, 1.0);
        const double len = std::hypot(1.0, slope);
        o.x = 1.0;
        o.y = camber_y(s, 1.0);
        o.nx = 1.0 / len;
        o.ny = slope / len;
        return o;
    }
    if (std::fabs(theta - M_PI) < 1e-14) {
        o.x = 0.0;
        o.y = 0.0;
        o.nx = -1.0;
        o.ny = 0.0;
        return o;
    }
    const double yt = half_thickness(s, xc);
    const double yc = camber_y(s, xc);
    const double dyc = camber_dx(s, xc);
    const double delta = std::atan(dyc);
    const double sd = std::sin(delta), cd = std::cos(delta);
    o.x = xc - side * yt * sd;
    o.y = yc + side * yt * cd;
    const double dyt = half_thickness_dx(s, xc);
    const double ddelta = camber_dxx(s, xc) / (1.0 + dyc * dyc);
    const double tx = 1.0 - side * (dyt * sd + yt * cd * ddelta);
    const double ty = dyc + side * (dyt * cd - yt * sd * ddelta);
    const double dir = upper ? -1.0 : 1.0;
    const double gx = dir * tx, gy = dir * ty;
    const double len = std::hypot(gx, gy);
    o.nx = gy / len;
    o.ny = -gx / len;
    return o;
}

// Bisection for the geometric stretch factor, pointcloud.cpp:152-168
double stretch_factor(int levels, double target)
{
    auto first_gap = [&](double sg) { return (sg - 1.0) / (std::pow(sg, levels) - 1.0); };
    double lo = 1.0 + 1e-9, hi = 3.0;
    if (first_gap(hi) > target) return hi;
    if (first_gap(lo) < target) return lo;
    for (int it = 0; it < 200; ++it) {
        const double mid = 0.5 * (lo + hi);
        if (first_gap(mid) > target)
            lo = mid;
        else
            hi = mid;
    }
    return 0.5 * (lo + hi);
}

struct Mom {
    double xx = 0.0, yy = 0.0, xy = 0.0;
};

Mom moments_of(const Cloud& c, int p, const int* st, int m)
{
    Mom r;
    for (int k = 0; k < m; ++k) {
        const double dx = c.x[st[k]] - c.x[p];
        const double dy = c.y[st[k]] - c.y[p];
        r.xx += dx * dx;
        r.yy += dy * dy;
        r.xy += dx * dy;
    }
    return r;
}

// classify_moments, spatial.cpp:29-38
int classify_moments(const Mom& m, int n)
{
    if (n == 0) return kEmpty;
    if (m.xx == 0.0 && m.yy == 0.0) return kSingular;
    if (m.yy == 0.0) return kLineX;
    if (m.xx == 0.0) return kLineY;
    const double det = m.xx * m.yy - m.xy * m.xy;
    if (det < kSingularDetEps * m.xx * m.yy) return kSingular;
    return kRegular;
}

// build_split_stencils' report predicate, pointcloud.cpp:264-277
bool report_singular(const Cloud& c, int p, const int* st, int m)
{
    if (m == 0) return false;
    const Mom r = moments_of(c, p, st, m);
    if (r.xx == 0.0 || r.yy == 0.0) return false;
    const double det = r.xx * r.yy - r.xy * r.xy;
    return det < kSingularDetEps * r.xx * r.yy;
}

void split_stencils(Cloud& c)
{
    // two passes (count, then fill) so every point is independent: the lists
    // and reports are exactly the sequential ones (pointcloud.cpp:257-299)
    const int n = c.n;
    auto in_slot = [&](int p, int q, int slot) {
        const double dx = c.x[q] - c.x[p];
        const double dy = c.y[q] - c.y[p];
        switch (slot) {
            case kXpos: return dx >= 0.0;
            case kXneg: return dx <= 0.0;
            case kYpos: return dy >= 0.0;
            default: return dy <= 0.0;
        }
    };
    for (int sl = 0; sl < 4; ++sl) {
        Csr& s = c.split[sl];
        fresh(s.off, n + 1, 0);
#pragma omp parallel for schedule(static)
        for (int p = 0; p < n; ++p) {
            int m = 0;
            for (int k = c.nbr.off[p]; k < c.nbr.off[p + 1]; ++k) m += in_slot(p, c.nbr.idx[k], sl);
            s.off[p + 1] = m;
        }
        for (int p = 0; p < n; ++p) s.off[p + 1] += s.off[p];
        s.idx.clear();
        s.idx.resize(s.off[n]);  // (every entry written below)
#pragma omp parallel for schedule(static)
        for (int p = 0; p < n; ++p) {
            int w = s.off[p];
            for (int k = c.nbr.off[p]; k < c.nbr.off[p + 1]; ++k)
                if (in_slot(p, c.nbr.idx[k], sl)) s.idx[w++] = c.nbr.idx[k];
        }
    }
    std::vector<char> empty(n, 0), singular(n, 0);
#pragma omp parallel for schedule(static)
    for (int p = 0; p < n; ++p) {
        bool any_empty = false, any_singular = false;
        for (auto& s : c.split) {
            const int m = s.off[p + 1] - s.off[p];
            any_empty = any_empty || m == 0;
            any_singular = any_singular || report_singular(c, p, s.idx.data() + s.off[p], m);
        }
        any_singular = any_singular ||
                       report_singular(c, p, c.nbr.idx.data() + c.nbr.off[p], c.nbr.degree(p));
        empty[p] = any_empty;
        singular[p] = any_singular;
    }
    c.empty_points.clear();
    c.singular_points.clear();
    for (int p = 0; p < n; ++p) {
        if (empty[p]) c.empty_points.push_back(p);
        if (singular[p]) c.singular_points.push_back(p);
    }
}

// fill_split, spatial.cpp:40-76. axis_x: weight along x, else y.
void split_weights(Cloud& c, int slot, bool axis_x, int p, bool& flagged)
{
    const Csr& s = c.split[slot];
    const int b = s.off[p], m = s.off[p + 1] - b;
    const int* st = s.idx.data() + b;
    double* w = c.split_w[slot].data() + b;
    for (int k = 0; k < m; ++k) w[k] = 0.0;
    const Mom mo = moments_of(c, p, st, m);
    const int cls = classify_moments(mo, m);
    c.split_class[slot][p] = cls;
    c.ls_one[slot][p] = 0.0;
    const int l = 2 + slot;
    c.coefA[l][p] = 0.0;
    c.coefB[l][p] = 0.0;
    c.coefD[l][p] = 1.0;
    if (cls == kLineX && axis_x) {
        c.coefA[l][p] = 1.0;
        c.coefD[l][p] = mo.xx;
    } else if (cls == kLineY && !axis_x) {
        c.coefA[l][p] = 1.0;
        c.coefD[l][p] = mo.yy;
    } else if (cls == kRegular) {
        c.coefA[l][p] = axis_x ? mo.yy : mo.xx;
        c.coefB[l][p] = mo.xy;
        c.coefD[l][p] = mo.xx * mo.yy - mo.xy * mo.xy;
    }
    if (cls == kEmpty) return;
    if (cls == kSingular) {
        flagged = true;
        return;
    }
    if (cls == kLineX) {
        if (!axis_x) return;
        for (int k = 0; k < m; ++k) w[k] = (c.x[st[k]] - c.x[p]) / mo.xx;
    } else if (cls == kLineY) {
        if (axis_x) return;
        for (int k = 0; k < m; ++k) w[k] = (c.y[st[k]] - c.y[p]) / mo.yy;
    } else {
        const double den = mo.xx * mo.yy - mo.xy * mo.xy;
        for (int k = 0; k < m; ++k) {
            const double dx = c.x[st[k]] - c.x[p];
            const double dy = c.y[st[k]] - c.y[p];
            w[k] = axis_x ? (mo.yy * dx - mo.xy * dy) / den : (mo.xx * dy - mo.xy * dx) / den;
        }
    }
    double sum = 0.0;
    for (int k = 0; k < m; ++k) sum += w[k];
    c.ls_one[slot][p] = sum;
}

void ls_operators(Cloud& c)
{
    const size_t nnz = c.nbr.idx.size();
    fresh(c.wx, nnz, 0.0);
    fresh(c.wy, nnz, 0.0);
    fresh(c.full_class, c.n, int(kEmpty));
    for (int s = 0; s < 4; ++s) {
        fresh(c.split_w[s], c.split[s].idx.size(), 0.0);
        fresh(c.ls_one[s], c.n, 0.0);
        fresh(c.split_class[s], c.n, int(kEmpty));
    }
    for (int l = 0; l < 6; ++l) {
        fresh(c.coefA[l], c.n, 0.0);
        fresh(c.coefB[l], c.n, 0.0);
        fresh(c.coefD[l], c.n, 1.0);
    }
    c.flagged.clear();
    std::vector<char> flags(c.n, 0);
#pragma omp parallel for schedule(static)
    for (int p = 0; p < c.n; ++p) {
        bool flagged = false;
        const int b = c.nbr.off[p], m = c.nbr.degree(p);
        const int* st = c.nbr.idx.data() + b;
        const Mom mo = moments_of(c, p, st, m);
        const int cls = classify_moments(mo, m);
        c.full_class[p] = cls;
        if (cls == kRegular) {
            const double den = mo.xx * mo.yy - mo.xy * mo.xy;
            c.coefA[0][p] = mo.yy;
            c.coefB[0][p] = mo.xy;
            c.coefD[0][p] = den;
            c.coefA[1][p] = mo.xx;
            c.coefB[1][p] = mo.xy;
            c.coefD[1][p] = den;
            for (int k = 0; k < m; ++k) {
                const double dx = c.x[st[k]] - c.x[p];
                const double dy = c.y[st[k]] - c.y[p];
                c.wx[b + k] = (mo.yy * dx - mo.xy * dy) / den;
                c.wy[b + k] = (mo.xx * dy - mo.xy * dx) / den;
            }
        } else if (cls == kLineX) {
            c.coefA[0][p] = 1.0;
            c.coefD[0][p] = mo.xx;
            for (int k = 0; k < m; ++k) c.wx[b + k] = (c.x[st[k]] - c.x[p]) / mo.xx;
        } else if (cls == kLineY) {
            c.coefA[1][p] = 1.0;
            c.coefD[1][p] = mo.yy;
            for (int k = 0; k < m; ++k) c.wy[b + k] = (c.y[st[k]] - c.y[p]) / mo.yy;
        } else if (cls == kSingular) {
            flagged = true;
        }
        split_weights(c, kXpos, true, p, flagged);
        split_weights(c, kXneg, true, p, flagged);
        split_weights(c, kYpos, false, p, flagged);
        split_weights(c, kYneg, false, p, flagged);
        flags[p] = flagged;
    }
    for (int p = 0; p < c.n; ++p)
        if (flags[p]) c.flagged.push_back(p);
}

// Greedy colouring over the symmetrised graph, coloring.cpp:7-52.
void greedy_colors(Cloud& c)
{
    // symmetrised adjacency (coloring.cpp:7-21): row i = nbr(i) then the
    // transpose entries, built in parallel (the transpose slots are taken
    // atomically; the order is irrelevant, every row is sorted below)
    const int n = c.n;
    std::vector<long> deg(n, 0);
#pragma omp parallel for schedule(static)
    for (int i = 0; i < n; ++i) deg[i] = c.nbr.degree(i);
#pragma omp parallel for schedule(static)
    for (int i = 0; i < n; ++i)
        for (int k = c.nbr.off[i]; k < c.nbr.off[i + 1]; ++k) __atomic_fetch_add(&deg[c.nbr.idx[k]], 1L, __ATOMIC_RELAXED);
    std::vector<long> aoff(n + 1, 0);
    for (int i = 0; i < n; ++i) aoff[i + 1] = aoff[i] + deg[i];
    bvec<int> adj;
    adj.resize(aoff[n]);  // (every entry written below)
    std::vector<long> pos(n);
#pragma omp parallel for schedule(static)
    for (int i = 0; i < n; ++i) {
        const int d = c.nbr.degree(i);
        std::copy(c.nbr.idx.data() + c.nbr.off[i], c.nbr.idx.data() + c.nbr.off[i] + d, adj.data() + aoff[i]);
        pos[i] = aoff[i] + d;
    }
#pragma omp parallel for schedule(static)
    for (int i = 0; i < n; ++i)
        for (int k = c.nbr.off[i]; k < c.nbr.off[i + 1]; ++k)
            adj[__atomic_fetch_add(&pos[c.nbr.idx[k]], 1L, __ATOMIC_RELAXED)] = i;
    std::vector<int> len(n);
#pragma omp parallel for schedule(static)
    for (int i = 0; i < n; ++i) {
        int* a = adj.data() + aoff[i];
        const int m = static_cast<int>(aoff[i + 1] - aoff[i]);
        std::sort(a, a + m);
        len[i] = static_cast<int>(std::unique(a, a + m) - a);
    }
    fresh(c.color, n, 0);
    if (n > 0) c.color[0] = 1;
    // the smallest colour no neighbour holds (the reference's `used` scan,
    // coloring.cpp:36-44): a 64-bit mask of colours 1..64, the reference's
    // scan only when all 64 are taken
    std::vector<char> seen;
    for (int i = 0; i < n; ++i) {
        for (int t = 0; t < len[i]; ++t) {
            const int p = adj[aoff[i] + t];
            if (c.color[p] != 0) continue;
            const int* ap = adj.data() + aoff[p];
            unsigned long long used = 0;
            for (int u = 0; u < len[p]; ++u) {
                const int cq = c.color[ap[u]];
                if (cq > 0 && cq <= 64) used |= 1ull << (cq - 1);
            }
            int k = __builtin_ffsll(static_cast<long long>(~used));
            if (k == 0) {
                seen.assign(static_cast<size_t>(len[p]) + 2, 0);
                for (int u = 0; u < len[p]; ++u) {
                    const int cq = c.color[ap[u]];
                    if (cq > 0 && cq < static_cast<int>(seen.size())) seen[cq] = 1;
                }
                k = 1;
                while (seen[k]) ++k;
            }
            c.color[p] = k;
        }
    }
    for (int i = 0; i < n; ++i)
        if (c.color[i] == 0) c.color[i] = 1;
    c.n_colors = n > 0 ? *std::max_element(c.color.begin(), c.color.end()) : 0;
}

// Minimal istream-like scanner over one line (pointcloud.cpp:310-356 reads
// each record with operator>>).
struct LineScanner {
    const char* s;
    bool get_long(long& v)
    {
        char* end = nullptr;
        errno = 0;
        const long r = std::strtol(s, &end, 10);
        if (end == s || errno == ERANGE) return false;
        v = r;
        s = end;
        return true;
    }
    bool get_int(int& v)
    {
        long t;
        if (!get_long(t) || t < std::numeric_limits<int>::min() ||
            t > std::numeric_limits<int>::max())
            return false;
        v = static_cast<int>(t);
        return true;
    }
    bool get_double(double& v)
    {
        char* end = nullptr;
        const double r = std::strtod(s, &end);
        if (end == s) return false;
        v = r;
        s = end;
        return true;
    }
};

}  // namespace

void finalize(Cloud& c)
{
    const bool tm = std::getenv("KF_TIME_INGEST") != nullptr;
    auto now = [] { return std::chrono::steady_clock::now(); };
    auto t0 = now();
    c.wall_ids.clear();
    c.interior_ids.clear();
    c.outer_ids.clear();
    for (int i = 0; i < c.n; ++i) {
        if (c.kind[i] == kWall) c.wall_ids.push_back(i);
        if (c.kind[i] == kInterior) c.interior_ids.push_back(i);
        if (c.kind[i] == kOuter) c.outer_ids.push_back(i);
    }
    auto t1 = now();
    // the greedy colouring reads only the neighbour lists: it runs on its own
    // thread (its scan is sequential, coloring.cpp:29-44) while the split
    // stencils and the LS operators are built
    std::exception_ptr col_err;
    double col_s = 0.0;
    std::thread col([&] {
        try {
            const auto a = now();
            greedy_colors(c);
            col_s = std::chrono::duration<double>(now() - a).count();
        } catch (...) {
            col_err = std::current_exception();
        }
    });
    auto t2 = t1, t3 = t1;
    try {
        split_stencils(c);
        t2 = now();
        ls_operators(c);
        t3 = now();
    } catch (...) {
        col.join();
        throw;
    }
    col.join();
    if (col_err) std::rethrow_exception(col_err);
    auto t4 = now();
    if (tm)
        std::fprintf(stderr, "ingest: lists %.2f split %.2f ls %.2f colour %.2f s (concurrent; %.2f s after the LS)\n",
                     std::chrono::duration<double>(t1 - t0).count(), std::chrono::duration<double>(t2 - t1).count(),
                     std::chrono::duration<double>(t3 - t2).count(), col_s, std::chrono::duration<double>(t4 - t3).count());
}

Cloud generate_naca_ogrid(const std::string& digits, int n_wall, int n_radial,
                          double far_field_radius)
{
    const Naca4 shape = parse_digits(digits);
    if (n_wall < 32 || n_radial < 8 || far_field_radius < 10.0)
        throw IngestError(1,
                          "degenerate O-grid parameters (need n_wall >= 32, n_radial >= 8, "
                          "far_field_radius >= 10)");
    const double cx = 0.5, cy = 0.0;
    const long N = static_cast<long>(n_wall) * n_radial;
    if (N > std::numeric_limits<int>::max() / 8)
        throw IngestError(1, "O-grid too large for 32-bit indexing");
    Cloud c;
    c.n = static_cast<int>(N);
    c.x.resize(N);
    c.y.resize(N);
    fresh(c.nx, N, 0.0);
    fresh(c.ny, N, 0.0);
    fresh(c.kind, N, int(kInterior));

    std::vector<WallSample> wall(n_wall);
    for (int i = 0; i < n_wall; ++i) wall[i] = surface_at(shape, 2.0 * M_PI * i / n_wall);
    double perimeter = 0.0;
    for (int i = 0; i < n_wall; ++i) {
        const WallSample& a = wall[i];
        const WallSample& b = wall[(i + 1) % n_wall];
        perimeter += std::hypot(b.x - a.x, b.y - a.y);
    }
    const double first_layer = perimeter / n_wall;
    const double mean_ray = far_field_radius - 0.5;
    const double sigma = stretch_factor(n_radial - 1, first_layer / mean_ray);
    std::vector<double> frac(n_radial);
    for (int j = 0; j < n_radial; ++j)
        frac[j] = (std::pow(sigma, j) - 1.0) / (std::pow(sigma, n_radial - 1) - 1.0);

#pragma omp parallel for schedule(static)
    for (int i = 0; i < n_wall; ++i) {
        const WallSample& s = wall[i];
        const double phi = std::atan2(s.y - cy, s.x - cx);
        const double fx = cx + far_field_radius * std::cos(phi);
        const double fy = cy + far_field_radius * std::sin(phi);
        for (int j = 0; j < n_radial; ++j) {
            const long id = static_cast<long>(j) * n_wall + i;
            c.x[id] = s.x + frac[j] * (fx - s.x);
            c.y[id] = s.y + frac[j] * (fy - s.y);
            if (j == 0) {
                c.kind[id] = kWall;
                c.nx[id] = s.nx;
                c.ny[id] = s.ny;
            } else if (j == n_radial - 1) {
                c.kind[id] = kOuter;
                c.nx[id] = std::cos(phi);
                c.ny[id] = std::sin(phi);
            }
        }
    }

    // Eight-neighbourhood, wrapped in i and clamped in j (pointcloud.cpp:237-250):
    // rows 0 and n_radial-1 have 5 neighbours, the others 8, in this order
    c.nbr.off.assign(N + 1, 0);
    for (long id = 0; id < N; ++id) {
        const int j = static_cast<int>(id / n_wall);
        c.nbr.off[id + 1] = c.nbr.off[id] + ((j == 0 || j == n_radial - 1) ? 5 : 8);
    }
    if (n_radial == 1) throw IngestError(1, "degenerate O-grid");
    c.nbr.idx.resize(c.nbr.off[N]);  // (every entry written below)
#pragma omp parallel for schedule(static)
    for (int j = 0; j < n_radial; ++j) {
        for (int i = 0; i < n_wall; ++i) {
            const long id = static_cast<long>(j) * n_wall + i;
            int w = c.nbr.off[id];
            for (int dj = -1; dj <= 1; ++dj) {
                const int jj = j + dj;
                if (jj < 0 || jj >= n_radial) continue;
                for (int di = -1; di <= 1; ++di) {
                    if (di == 0 && dj == 0) continue;
                    const int ii = (i + di + n_wall) % n_wall;
                    c.nbr.idx[w++] = jj * n_wall + ii;
                }
            }
        }
    }
    finalize(c);
    return c;
}

Cloud cloud_from_arrays(int n, const double* x, const double* y, const int* kind,
                        const double* nx, const double* ny, const int* off, const int* idx)
{
    if (n < 0) throw IngestError(1, "negative point count");
    Cloud c;
    c.n = n;
    c.x.assign(x, x + n);
    c.y.assign(y, y + n);
    c.nx.assign(nx, nx + n);
    c.ny.assign(ny, ny + n);
    c.kind.assign(kind, kind + n);
    c.nbr.off.assign(off, off + n + 1);
    if (off[0] != 0) throw IngestError(1, "neighbour offsets must start at 0");
    for (int p = 0; p < n; ++p) {
        if (off[p + 1] < off[p]) throw IngestError(1, "neighbour offsets must be nondecreasing");
        if (kind[p] < 0 || kind[p] > 2) throw IngestError(1, "bad point kind at point " + std::to_string(p));
    }
    c.nbr.idx.assign(idx, idx + off[n]);
    for (int q : c.nbr.idx)
        if (q < 0 || q >= n) throw IngestError(1, "neighbour id out of range");
    finalize(c);
    return c;
}

// Binary SoA cloud cache: "KFCLOUD1", n, nnz (int64),
// then x, y, nx, ny (n doubles each), kind (n int32), offsets (n+1 int32),
// neighbour ids (nnz int32, 0-based). Read with a few bulk reads instead of
// a line parser; the same validation as the array path (cloud_from_arrays).
static const char kBinMagic[8] = {'K', 'F', 'C', 'L', 'O', 'U', 'D', '1'};

static Cloud load_cloud_binary(const std::string& path)
{
    std::FILE* f = std::fopen(path.c_str(), "rb");
    if (!f) throw IngestError(2, "cannot open cloud file: " + path);
    auto rd = [&](void* p, size_t bytes) {
        if (bytes && std::fread(p, 1, bytes, f) != bytes) {
            std::fclose(f);
            throw IngestError(2, path + ": truncated binary cloud");
        }
    };
    char magic[8];
    rd(magic, 8);
    long long hdr[2];
    rd(hdr, sizeof hdr);
    const long long n = hdr[0], nnz = hdr[1];
    if (n <= 0 || n > (1ll << 31) - 2 || nnz < 0 || nnz > (1ll << 31) - 1) {
        std::fclose(f);
        throw IngestError(2, path + ": bad binary cloud header");
    }
    std::vector<double> x(n), y(n), nx(n), ny(n);
    std::vector<int> kind(n), off(n + 1), idx(nnz);
    rd(x.data(), 8 * n);
    rd(y.data(), 8 * n);
    rd(nx.data(), 8 * n);
    rd(ny.data(), 8 * n);
    rd(kind.data(), 4 * n);
    rd(off.data(), 4 * (n + 1));
    rd(idx.data(), 4 * nnz);
    std::fclose(f);
    if (off[n] != nnz) throw IngestError(2, path + ": neighbour offsets do not match the entry count");
    return cloud_from_arrays(static_cast<int>(n), x.data(), y.data(), kind.data(), nx.data(), ny.data(),
                             off.data(), idx.data());
}

void save_cloud_binary(const Cloud& c, const std::string& path)
{
    std::FILE* f = std::fopen(path.c_str(), "wb");
    if (!f) throw IngestError(2, "cannot write cloud file: " + path);
    const long long hdr[2] = {c.n, static_cast<long long>(c.nbr.idx.size())};
    bool ok = std::fwrite(kBinMagic, 1, 8, f) == 8 && std::fwrite(hdr, sizeof hdr, 1, f) == 1;
    auto wr = [&](const void* p, size_t bytes) {
        if (ok && bytes) ok = std::fwrite(p, 1, bytes, f) == bytes;
    };
    wr(c.x.data(), 8 * c.x.size());
    wr(c.y.data(), 8 * c.y.size());
    wr(c.nx.data(), 8 * c.nx.size());
    wr(c.ny.data(), 8 * c.ny.size());
    std::vector<int> kind(c.kind.begin(), c.kind.end());
    wr(kind.data(), 4 * kind.size());
    wr(c.nbr.off.data(), 4 * c.nbr.off.size());
    wr(c.nbr.idx.data(), 4 * c.nbr.idx.size());
    ok = (std::fclose(f) == 0) && ok;
    if (!ok) throw IngestError(2, "cannot write cloud file: " + path);
}

static Cloud load_cloud_text(const std::string& path);

Cloud load_cloud(const std::string& path)
{
    {
        // the binary cache is recognised by its magic; anything else is the
        // reference's text format
        std::FILE* f = std::fopen(path.c_str(), "rb");
        char magic[8] = {0};
        const bool bin = f && std::fread(magic, 1, 8, f) == 8 && std::memcmp(magic, kBinMagic, 8) == 0;
        if (f) std::fclose(f);
        if (bin) return load_cloud_binary(path);
    }
    return load_cloud_text(path);
}

// The reference's text format (load_cloud, pointcloud.cpp:301-381), parsed in
// parallel: the file is read whole, its lines are NUL-terminated in place
// (so a record's fields can never run into the next line) and split into
// contiguous per-thread ranges of records; every thread parses its records
// into its own CSR block, and the blocks are concatenated. Errors keep the
// reference's semantics: the first failing line in file order wins (each
// thread stops at its first failure; the smallest line number is reported),
// a count mismatch is reported only if no line failed, and the post-parse
// validation reports the smallest failing point.
static Cloud load_cloud_text(const std::string& path)
{
    std::FILE* f = std::fopen(path.c_str(), "rb");
    if (!f) throw IngestError(2, "cannot open cloud file: " + path);
    std::fseek(f, 0, SEEK_END);
    const long long size = std::ftell(f);
    std::fseek(f, 0, SEEK_SET);
    if (size < 0) {
        std::fclose(f);
        throw IngestError(2, "cannot open cloud file: " + path);
    }
    std::vector<char> buf(static_cast<size_t>(size) + 1);
    const bool rd_ok = size == 0 || std::fread(buf.data(), 1, size, f) == static_cast<size_t>(size);
    std::fclose(f);
    if (!rd_ok) throw IngestError(2, "cannot open cloud file: " + path);
    buf[size] = '\n';  // (sentinel: the last line needs no newline, as with getline)
    // ---- line starts (parallel newline scan; newlines become NULs)
    const int nt = std::max(1, omp_get_max_threads());
    std::vector<std::vector<long long>> nl(nt);
#pragma omp parallel num_threads(nt)
    {
        const int t = omp_get_thread_num();
        const long long lo = size * t / nt, hi = size * (t + 1) / nt;
        for (long long k = lo; k < hi; ++k)
            if (buf[k] == '\n') {
                nl[t].push_back(k);
                buf[k] = '\0';
            }
    }
    std::vector<long long> start(1, 0);
    for (auto& v : nl)
        for (long long k : v) start.push_back(k + 1);
    if (start.back() >= size) start.pop_back();  // no empty line after a final newline
    buf[size] = '\0';
    const long long n_lines = static_cast<long long>(start.size());
    // content lines (not blank, not a comment), in file order
    auto content = [&](long long l) {
        const char* q = buf.data() + start[l];
        while (*q == ' ' || *q == '\t' || *q == '\r') ++q;
        return *q != '\0' && *q != '#';
    };
    long long hdr = 0;
    while (hdr < n_lines && !content(hdr)) ++hdr;
    if (hdr == n_lines) throw IngestError(2, path + ": empty cloud file");
    long expected = -1;
    {
        LineScanner sc{buf.data() + start[hdr]};
        if (!sc.get_long(expected) || expected <= 0)
            throw IngestError(2, path + ":" + std::to_string(hdr + 1) + ": parse error: bad point count header");
    }
    std::vector<long long> rec;  // line index of each record
    {
        std::vector<char> isrec(n_lines, 0);
#pragma omp parallel for schedule(static)
        for (long long l = hdr + 1; l < n_lines; ++l) isrec[l] = content(l) ? 1 : 0;
        rec.reserve(static_cast<size_t>(std::max(expected, 1L)));
        for (long long l = hdr + 1; l < n_lines; ++l)
            if (isrec[l]) rec.push_back(l);
    }
    const long long n_rec = static_cast<long long>(rec.size());
    if (n_rec > std::numeric_limits<int>::max() / 2)
        throw IngestError(2, path + ": too many points for 32-bit indexing");
    Cloud c;
    c.x.resize(n_rec);
    c.y.resize(n_rec);
    c.nx.assign(n_rec, 0.0);
    c.ny.assign(n_rec, 0.0);
    c.kind.assign(n_rec, 0);
    c.nbr.off.assign(n_rec + 1, 0);
    std::vector<std::vector<int>> ids(nt);
    std::vector<long long> err_line(nt, std::numeric_limits<long long>::max());
    std::vector<std::string> err_msg(nt);
#pragma omp parallel num_threads(nt)
    {
        const int t = omp_get_thread_num();
        const long long lo = n_rec * t / nt, hi = n_rec * (t + 1) / nt;
        std::vector<int>& out = ids[t];
        out.reserve(static_cast<size_t>((hi - lo) * 8));
        for (long long r = lo; r < hi; ++r) {
            const long long l = rec[r];
            auto fail = [&](const std::string& why) {
                err_line[t] = l + 1;
                err_msg[t] = path + ":" + std::to_string(l + 1) + ": parse error: " + why;
            };
            LineScanner sc{buf.data() + start[l]};
            long pid;
            double px, py;
            int kd, nn;
            if (!(sc.get_long(pid) && sc.get_double(px) && sc.get_double(py) && sc.get_int(kd) &&
                  sc.get_int(nn))) {
                fail("bad point record");
                break;
            }
            if (pid != r + 1) {
                fail("point index " + std::to_string(pid) + " out of order");
                break;
            }
            if (kd < 0 || kd > 2) {
                fail("bad point kind " + std::to_string(kd));
                break;
            }
            if (nn < 0) {
                fail("negative neighbour count");
                break;
            }
            bool ok = true;
            for (int k = 0; k < nn; ++k) {
                long v;
                if (!sc.get_long(v)) {
                    fail("missing neighbour id");
                    ok = false;
                    break;
                }
                out.push_back(static_cast<int>(v - 1));
            }
            if (!ok) break;
            double vx = 0.0, vy = 0.0;
            if ((kd == kWall || kd == kOuter) && !(sc.get_double(vx) && sc.get_double(vy))) {
                fail("missing normal for boundary point");
                break;
            }
            c.x[r] = px;
            c.y[r] = py;
            c.kind[r] = kd;
            c.nx[r] = vx;
            c.ny[r] = vy;
            c.nbr.off[r + 1] = nn;
        }
    }
    {
        int first = 0;
        for (int t = 1; t < nt; ++t)
            if (err_line[t] < err_line[first]) first = t;
        if (err_line[first] != std::numeric_limits<long long>::max()) throw IngestError(2, err_msg[first]);
    }
    if (n_rec != expected)
        throw IngestError(2, path + ": expected " + std::to_string(expected) + " points, found " +
                                 std::to_string(n_rec));
    for (long long r = 0; r < n_rec; ++r) {
        c.nbr.off[r + 1] += c.nbr.off[r];
        if (c.nbr.off[r + 1] < 0) throw IngestError(2, path + ": too many neighbour entries for 32-bit offsets");
    }
    c.nbr.idx.resize(c.nbr.off[n_rec]);
#pragma omp parallel num_threads(nt)
    {
        const int t = omp_get_thread_num();
        const long long lo = n_rec * t / nt;
        std::copy(ids[t].begin(), ids[t].end(), c.nbr.idx.begin() + c.nbr.off[lo]);
    }
    c.n = static_cast<int>(n_rec);
    // post-parse validation in point order (pointcloud.cpp:357-376): the
    // smallest failing point wins
    int bad = c.n;
    std::string bad_msg;
#pragma omp parallel for schedule(static) reduction(min : bad)
    for (int i = 0; i < c.n; ++i) {
        bool b = c.nbr.degree(i) < 3;
        for (int k = c.nbr.off[i]; k < c.nbr.off[i + 1] && !b; ++k) {
            const int q = c.nbr.idx[k];
            b = q < 0 || q >= c.n || q == i;
        }
        if (!b && c.kind[i] != kInterior) b = std::fabs(std::hypot(c.nx[i], c.ny[i]) - 1.0) > 1e-6;
        if (b) bad = std::min(bad, i);
    }
    // the failing point's checks in the reference's order, for its message
    if (bad < c.n) {
        const int i = bad;
        if (c.nbr.degree(i) < 3)
            throw IngestError(2, path + ": point " + std::to_string(i + 1) +
                                     " has fewer than 3 neighbours");
        for (int k = c.nbr.off[i]; k < c.nbr.off[i + 1]; ++k) {
            const int q = c.nbr.idx[k];
            if (q < 0 || q >= c.n)
                throw IngestError(2, path + ": point " + std::to_string(i + 1) +
                                         " has out-of-range neighbour " + std::to_string(q + 1));
            if (q == i)
                throw IngestError(2, path + ": point " + std::to_string(i + 1) +
                                         " lists itself as neighbour");
        }
        if (c.kind[i] != kInterior) {
            const double len = std::hypot(c.nx[i], c.ny[i]);
            if (std::fabs(len - 1.0) > 1e-6)
                throw IngestError(2, path + ": point " + std::to_string(i + 1) +
                                         " has a non-unit normal");
        }
    }
    finalize(c);
    return c;
}

void save_cloud(const Cloud& c, const std::string& path)
{
    std::FILE* f = std::fopen(path.c_str(), "w");
    if (!f) throw IngestError(2, "cannot write cloud file: " + path);
    std::fprintf(f, "%d\n", c.n);
    for (int i = 0; i < c.n; ++i) {
        std::fprintf(f, "%d %.17g %.17g %d %d", i + 1, c.x[i], c.y[i], c.kind[i], c.nbr.degree(i));
        for (int k = c.nbr.off[i]; k < c.nbr.off[i + 1]; ++k) std::fprintf(f, " %d", c.nbr.idx[k] + 1);
        if (c.kind[i] != kInterior) std::fprintf(f, " %.17g %.17g", c.nx[i], c.ny[i]);
        std::fputc('\n', f);
    }
    std::fclose(f);
}

}  // namespace kfb
