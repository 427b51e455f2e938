// Spatial domain decomposition of a point cloud across ranks (SURVEY.md
// §8(e)) and the local numbering of one rank, host-side C++.
//
// Every stage of an iteration reads only 1-ring neighbours (the full
// stencil `nbr` and its split subsets), so a rank owns a set of points and
// holds read-only copies ("ghosts") of the non-owned neighbours of its owned
// points. The outer boundary condition copies the updated state of an
// outer point's nearest interior neighbour (driver.cpp:51-65,85-94); the
// planner gives each outer point to the owner of that neighbour, so the BC
// never needs a remote value.
//
// Local numbering (colour-major like the single-GPU layout, so the sweep's
// "lower colour" test stays an index compare): for each colour c
//   [gs[c], oe[c])  owned points of colour c (in-colour order as 1 GPU),
//                   padded to a multiple of 32;
//   [oe[c], ge[c])  ghosts of colour c grouped by owning peer (ascending
//                   rank), ascending global id inside a peer, padded to 32.
// A rank sends to peer s, per colour, its owned points that are ghosts of s,
// in ascending global id: exactly the order s stores them in, so a message
// lands contiguously in s's ghost range.
#pragma once

#include <cstdint>
#include <vector>

#include "cloud.hpp"

namespace kfb {

// Morton code of every point over the cloud's bounding box (32 bits/axis).
std::vector<uint64_t> morton_codes(const Cloud& c);

enum PartitionMode : int { kPartAngular = 0, kPartMorton = 1 };

// owner[p] in [0, n_parts) for every point, equal-count chunks of the
// angular (about the wall centroid) or Morton order, then outer points moved
// to the owner of their BC source.
std::vector<int> plan_partition(const Cloud& c, int n_parts, int mode);

// Nearest interior neighbour of each point (first minimum in nbr order,
// driver.cpp:51-65), or -1; the outer BC source.
std::vector<int> bc_sources(const Cloud& c);

struct LocalLayout {
    int rank = 0, n_parts = 1, n_colors = 1;
    std::vector<int> perm;           // local -> global (-1 = padding)
    std::vector<unsigned char> ghost;  // local index is a ghost copy
    std::vector<int> gs, oe, ge;     // per colour: block start, owned end, block end
    // per colour: end of the boundary owned points (gs <= ob <= oe). Owned
    // points a peer holds as ghosts come first in their colour block, so the
    // solver can update them, start their halo exchange and update the
    // interior [ob, oe) while it is in flight.
    std::vector<int> ob;
    std::vector<int> peers;          // ranks exchanged with, ascending
    // per peer (index into peers) and colour
    std::vector<std::vector<int>> recv_off, recv_cnt;  // local ghost ranges
    std::vector<std::vector<std::vector<int>>> send_idx;  // local indices, ascending global id
    int n_owned = 0;
};

// Reverse Cuthill-McKee rank of every point (bandwidth-reducing order of the
// symmetrised stencil graph).
std::vector<int> rcm_rank(const Cloud& c);

// ordering: 0 natural (ascending global id), 2 reverse Cuthill-McKee,
// 1 Morton over the global
// bounding box (the single-GPU in-colour orders).
LocalLayout build_local_layout(const Cloud& c, const std::vector<int>& owner, int n_parts, int rank,
                               int ordering, const std::vector<uint64_t>* morton = nullptr);
// ids (ascending or not) reordered stably by key[id], in parallel
void sort_by_key(std::vector<int>& ids, const std::vector<uint64_t>& key);

}  // namespace kfb
