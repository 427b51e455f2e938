// Domain decomposition and local numbering (partition.hpp).
#include "partition.hpp"

#include <algorithm>
#include <parallel/algorithm>
#include <utility>
#include <cmath>
#include <cstdint>
#include <limits>
#include <numeric>
#include <stdexcept>
#include <string>

namespace kfb {

namespace {

uint64_t spread(uint64_t v)
{
    v &= 0xffffffffull;
    v = (v | (v << 16)) & 0x0000ffff0000ffffull;
    v = (v | (v << 8)) & 0x00ff00ff00ff00ffull;
    v = (v | (v << 4)) & 0x0f0f0f0f0f0f0f0full;
    v = (v | (v << 2)) & 0x3333333333333333ull;
    v = (v | (v << 1)) & 0x5555555555555555ull;
    return v;
}

}  // namespace

std::vector<uint64_t> morton_codes(const Cloud& c)
{
    std::vector<uint64_t> code(c.n, 0);
    if (c.n == 0) return code;
    const double x0 = *std::min_element(c.x.begin(), c.x.end());
    const double x1 = *std::max_element(c.x.begin(), c.x.end());
    const double y0 = *std::min_element(c.y.begin(), c.y.end());
    const double y1 = *std::max_element(c.y.begin(), c.y.end());
    const double sx = x1 > x0 ? 4294967295.0 / (x1 - x0) : 0.0;
    const double sy = y1 > y0 ? 4294967295.0 / (y1 - y0) : 0.0;
#pragma omp parallel for schedule(static)
    for (int p = 0; p < c.n; ++p)
        code[p] = spread(static_cast<uint32_t>((c.x[p] - x0) * sx)) |
                  (spread(static_cast<uint32_t>((c.y[p] - y0) * sy)) << 1);
    return code;
}

void sort_by_key(std::vector<int>& ids, const std::vector<uint64_t>& key)
{
    // stable by key for ascending ids == lexicographic (key, id)
    std::vector<std::pair<uint64_t, int>> kv(ids.size());
#pragma omp parallel for schedule(static)
    for (long long k = 0; k < static_cast<long long>(ids.size()); ++k) kv[k] = {key[ids[k]], ids[k]};
    if (!std::is_sorted(ids.begin(), ids.end())) {
        std::stable_sort(kv.begin(), kv.end(), [](const auto& a, const auto& b) { return a.first < b.first; });
    } else {
        __gnu_parallel::sort(kv.begin(), kv.end());
    }
#pragma omp parallel for schedule(static)
    for (long long k = 0; k < static_cast<long long>(ids.size()); ++k) ids[k] = kv[k].second;
}

std::vector<int> rcm_rank(const Cloud& c)
{
    // reverse Cuthill-McKee over the symmetrised stencil graph: breadth-first
    // from a minimum-degree start of every component, neighbours visited in
    // ascending degree (ties: id), the whole visit order reversed
    const int n = c.n;
    std::vector<int> deg(n, 0);
    for (int p = 0; p < n; ++p)
        for (int k = c.nbr.off[p]; k < c.nbr.off[p + 1]; ++k) {
            ++deg[p];
            ++deg[c.nbr.idx[k]];
        }
    std::vector<long> off(n + 1, 0);
    for (int p = 0; p < n; ++p) off[p + 1] = off[p] + deg[p];
    std::vector<int> adj(off[n]);
    std::vector<long> pos(off.begin(), off.end() - 1);
    for (int p = 0; p < n; ++p)
        for (int k = c.nbr.off[p]; k < c.nbr.off[p + 1]; ++k) {
            const int q = c.nbr.idx[k];
            adj[pos[p]++] = q;
            adj[pos[q]++] = p;
        }
    std::vector<int> order;
    order.reserve(n);
    std::vector<char> seen(n, 0);
    std::vector<int> by_deg(n);
    std::iota(by_deg.begin(), by_deg.end(), 0);
    std::stable_sort(by_deg.begin(), by_deg.end(), [&](int a, int b) { return deg[a] < deg[b]; });
    std::vector<int> nb;
    for (int start : by_deg) {
        if (seen[start]) continue;
        size_t head = order.size();
        order.push_back(start);
        seen[start] = 1;
        while (head < order.size()) {
            const int p = order[head++];
            nb.clear();
            for (long k = off[p]; k < off[p + 1]; ++k)
                if (!seen[adj[k]]) {
                    seen[adj[k]] = 1;
                    nb.push_back(adj[k]);
                }
            std::sort(nb.begin(), nb.end(), [&](int a, int b) { return deg[a] != deg[b] ? deg[a] < deg[b] : a < b; });
            order.insert(order.end(), nb.begin(), nb.end());
        }
    }
    std::vector<int> rank(n, 0);
    for (int k = 0; k < n; ++k) rank[order[n - 1 - k]] = k;
    return rank;
}

std::vector<int> bc_sources(const Cloud& c)
{
    std::vector<int> src(c.n, -1);
    for (int p = 0; p < c.n; ++p) {
        double best_d = std::numeric_limits<double>::max();
        for (int k = c.nbr.off[p]; k < c.nbr.off[p + 1]; ++k) {
            const int i = c.nbr.idx[k];
            const double d = std::hypot(c.x[i] - c.x[p], c.y[i] - c.y[p]);
            if (c.kind[i] == kInterior && d < best_d) {
                best_d = d;
                src[p] = i;
            }
        }
    }
    return src;
}

std::vector<int> plan_partition(const Cloud& c, int n_parts, int mode)
{
    if (n_parts < 1) throw std::invalid_argument("n_parts must be >= 1");
    std::vector<int> owner(c.n, 0);
    if (n_parts == 1 || c.n == 0) return owner;
    std::vector<int> order(c.n);
    std::iota(order.begin(), order.end(), 0);
    if (mode == kPartAngular) {
        double xc = 0.0, yc = 0.0;
        if (!c.wall_ids.empty()) {
            for (int p : c.wall_ids) {
                xc += c.x[p];
                yc += c.y[p];
            }
            xc /= static_cast<double>(c.wall_ids.size());
            yc /= static_cast<double>(c.wall_ids.size());
        } else {
            xc = 0.5 * (*std::min_element(c.x.begin(), c.x.end()) + *std::max_element(c.x.begin(), c.x.end()));
            yc = 0.5 * (*std::min_element(c.y.begin(), c.y.end()) + *std::max_element(c.y.begin(), c.y.end()));
        }
        std::vector<double> th(c.n);
        for (int p = 0; p < c.n; ++p) th[p] = std::atan2(c.y[p] - yc, c.x[p] - xc);
        std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return th[a] < th[b]; });
    } else if (mode == kPartMorton) {
        const std::vector<uint64_t> code = morton_codes(c);
        std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return code[a] < code[b]; });
    } else {
        throw std::invalid_argument("unknown partition mode " + std::to_string(mode));
    }
    for (int k = 0; k < c.n; ++k)
        owner[order[k]] = static_cast<int>(static_cast<long long>(k) * n_parts / c.n);
    // outer points follow their BC source (driver.cpp:85-94 reads it)
    const std::vector<int> src = bc_sources(c);
    for (int p = 0; p < c.n; ++p)
        if (c.kind[p] == kOuter && src[p] >= 0) owner[p] = owner[src[p]];
    return owner;
}

LocalLayout build_local_layout(const Cloud& c, const std::vector<int>& owner, int n_parts, int rank,
                               int ordering, const std::vector<uint64_t>* morton)
{
    if (static_cast<int>(owner.size()) != c.n) throw std::invalid_argument("owner size mismatch");
    if (rank < 0 || rank >= n_parts) throw std::invalid_argument("rank out of range");
    LocalLayout L;
    L.rank = rank;
    L.n_parts = n_parts;
    const int C = std::max(c.n_colors, 1);
    L.n_colors = C;
    auto col = [&](int p) { return std::max(c.color[p], 1) - 1; };

    // ghosts of every rank: non-owned neighbours of its owned points
    // is_ghost_of[s] as sorted unique lists is only needed for s == rank and
    // for the send lists (points of `rank` that are ghosts of s)
    std::vector<std::vector<int>> send_to(n_parts);  // global ids owned here, ghost of s
    std::vector<int> my_ghosts;
    if (n_parts > 1) {  // (one partition: no ghosts, nothing to send)
        for (int q = 0; q < c.n; ++q) {
            const int s = owner[q];
            for (int k = c.nbr.off[q]; k < c.nbr.off[q + 1]; ++k) {
                const int i = c.nbr.idx[k];
                const int oi = owner[i];
                if (oi == s) continue;
                if (s == rank) {
                    my_ghosts.push_back(i);
                } else if (oi == rank) {
                    send_to[s].push_back(i);
                }
            }
        }
        auto uniq = [](std::vector<int>& v) {
            std::sort(v.begin(), v.end());
            v.erase(std::unique(v.begin(), v.end()), v.end());
        };
        uniq(my_ghosts);
        for (auto& v : send_to) uniq(v);
    }

    // in-colour order of owned points (the single-GPU orders)
    std::vector<std::vector<int>> owned(C);
    {
        std::vector<int> cnt(C, 0);
        for (int p = 0; p < c.n; ++p)
            if (owner[p] == rank) ++cnt[col(p)];
        for (int cc = 0; cc < C; ++cc) owned[cc].reserve(cnt[cc]);
    }
    for (int p = 0; p < c.n; ++p)
        if (owner[p] == rank) owned[col(p)].push_back(p);
    if (ordering == 2) {
        const std::vector<int> rk = rcm_rank(c);
        for (auto& m : owned)
            std::stable_sort(m.begin(), m.end(), [&](int a, int b) { return rk[a] < rk[b]; });
    } else if (ordering == 1) {
        std::vector<uint64_t> own_code;
        if (!morton) own_code = morton_codes(c);
        const std::vector<uint64_t>& code = morton ? *morton : own_code;
        for (auto& m : owned) sort_by_key(m, code);
    }
    // boundary first inside every colour (stable: the chosen order within
    // each part). Boundary = sent to a peer OR reading a ghost (stencils
    // need not be symmetric): the interior neither feeds nor reads the halo.
    {
        std::vector<char> sent(c.n, 0);
        for (const auto& v : send_to)
            for (int g : v) sent[g] = 1;
        if (n_parts > 1)
#pragma omp parallel for schedule(static)
            for (int p = 0; p < c.n; ++p)
                if (owner[p] == rank)
                    for (int k = c.nbr.off[p]; k < c.nbr.off[p + 1] && !sent[p]; ++k)
                        if (owner[c.nbr.idx[k]] != rank) sent[p] = 1;
        for (auto& m : owned) std::stable_partition(m.begin(), m.end(), [&](int p) { return sent[p] != 0; });
        L.ob.assign(C, 0);
        for (int cc = 0; cc < C; ++cc) {
            int nb = 0;
            for (int p : owned[cc]) nb += sent[p];
            L.ob[cc] = nb;  // (made absolute below)
        }
    }
    // peers
    std::vector<int> is_peer(n_parts, 0);
    for (int g : my_ghosts) is_peer[owner[g]] = 1;
    for (int s = 0; s < n_parts; ++s)
        if (!send_to[s].empty()) is_peer[s] = 1;
    std::vector<int> peer_slot(n_parts, -1);
    for (int s = 0; s < n_parts; ++s)
        if (is_peer[s] && s != rank) {
            peer_slot[s] = static_cast<int>(L.peers.size());
            L.peers.push_back(s);
        }
    const int NP = static_cast<int>(L.peers.size());
    L.recv_off.assign(NP, std::vector<int>(C, 0));
    L.recv_cnt.assign(NP, std::vector<int>(C, 0));
    L.send_idx.assign(NP, std::vector<std::vector<int>>(C));
    // ghosts per colour, grouped by peer then ascending id (my_ghosts is
    // sorted by id already)
    std::vector<std::vector<std::vector<int>>> gh(C, std::vector<std::vector<int>>(NP));
    for (int g : my_ghosts) gh[col(g)][peer_slot[owner[g]]].push_back(g);

    L.gs.assign(C, 0);
    L.oe.assign(C, 0);
    L.ge.assign(C, 0);
    std::vector<int> inv(c.n, -1);
    {
        size_t cap = my_ghosts.size() + 64 * static_cast<size_t>(C) + 32;
        for (const auto& m : owned) cap += m.size();
        L.perm.reserve(cap);
        L.ghost.reserve(cap);
    }
    for (int cc = 0; cc < C; ++cc) {
        L.gs[cc] = static_cast<int>(L.perm.size());
        L.ob[cc] += L.gs[cc];
        for (int p : owned[cc]) {
            inv[p] = static_cast<int>(L.perm.size());
            L.perm.push_back(p);
            L.ghost.push_back(0);
            ++L.n_owned;
        }
        while (L.perm.size() % 32) {
            L.perm.push_back(-1);
            L.ghost.push_back(0);
        }
        L.oe[cc] = static_cast<int>(L.perm.size());
        for (int k = 0; k < NP; ++k) {
            L.recv_off[k][cc] = static_cast<int>(L.perm.size());
            L.recv_cnt[k][cc] = static_cast<int>(gh[cc][k].size());
            for (int g : gh[cc][k]) {
                inv[g] = static_cast<int>(L.perm.size());
                L.perm.push_back(g);
                L.ghost.push_back(1);
            }
        }
        while (L.perm.size() % 32) {
            L.perm.push_back(-1);
            L.ghost.push_back(0);
        }
        L.ge[cc] = static_cast<int>(L.perm.size());
    }
    if (L.perm.empty()) {
        for (int k = 0; k < 32; ++k) {
            L.perm.push_back(-1);
            L.ghost.push_back(0);
        }
        if (C > 0) L.oe[C - 1] = L.ge[C - 1] = 32;
        for (int cc = 0; cc < C; ++cc) L.ob[cc] = L.gs[cc];
    }
    for (int s = 0; s < n_parts; ++s) {
        if (peer_slot[s] < 0) continue;
        for (int g : send_to[s]) L.send_idx[peer_slot[s]][col(g)].push_back(inv[g]);
    }
    return L;
}

}  // namespace kfb
