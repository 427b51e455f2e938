// Host-side point-cloud ingestion for the B200 solver.
//
// Produces the same cloud, split stencils, least-squares weights and greedy
// colouring as the reference (bit-for-bit; tests/test_ingestion.py checks it)
// but stores everything as flat CSR arrays instead of vector-of-vectors, ready
// for the device packing in solver.cu. Reference counterparts:
//   generate_naca_ogrid   pointcloud.cpp:180-255
//   load_cloud/save_cloud pointcloud.cpp:301-401
//   build_split_stencils  pointcloud.cpp:257-299
//   build_ls_coefficients spatial.cpp:80-128
//   color_points          coloring.cpp:7-62
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "hostmem.hpp"

namespace kfb {

enum PointKindCode : int { kWall = 0, kInterior = 1, kOuter = 2 };
enum StencilClass : int { kRegular = 0, kLineX = 1, kLineY = 2, kEmpty = 3, kSingular = 4 };

// Split-list slot order used everywhere in this library (pointcloud.hpp:36).
enum SplitSlot : int { kXpos = 0, kXneg = 1, kYpos = 2, kYneg = 3 };

struct Csr {
    bvec<int> off;  // n+1
    bvec<int> idx;
    int degree(int p) const { return off[p + 1] - off[p]; }
};

struct Cloud {
    int n = 0;
    bvec<double> x, y, nx, ny;
    bvec<int> kind;
    Csr nbr;
    Csr split[4];  // xpos, xneg, ypos, yneg (same order as nbr within each list)

    // Least-squares operators (LsCoefficients, spatial.hpp:44-57).
    bvec<double> wx, wy;        // per nbr entry
    bvec<int> full_class;       // per point
    bvec<double> split_w[4];    // per split entry
    bvec<double> ls_one[4];     // per point
    bvec<int> split_class[4];   // per point
    std::vector<int> flagged;          // points owning a Singular stencil
    // The same weights as per-point linear forms of the entry offset, so the
    // device can rebuild them from gathered coordinates instead of streaming
    // them per entry: list l (0 full-x, 1 full-y, 2+slot split) gives
    //   x-form (l = 0, 2+kXpos, 2+kXneg): w = (A*dx - B*dy) / D
    //   y-form (l = 1, 2+kYpos, 2+kYneg): w = (A*dy - B*dx) / D
    // which is the reference's expression term for term (spatial.cpp:64-73,
    // 102-115), hence bitwise the stored weight; lists with no weights have
    // A = B = 0, D = 1.
    bvec<double> coefA[6], coefB[6], coefD[6];

    // StencilReport (pointcloud.hpp:21-26)
    std::vector<int> empty_points, singular_points;

    // Greedy colouring (1-based), n_colors.
    bvec<int> color;
    int n_colors = 0;

    std::vector<int> wall_ids, interior_ids, outer_ids;
};

struct IngestError : std::runtime_error {
    int kind;  // 1 invalid argument, 2 runtime (parse / io / invariant)
    IngestError(int k, const std::string& m) : std::runtime_error(m), kind(k) {}
};

// Raw constructors: fill geometry + nbr, then call finalize().
Cloud generate_naca_ogrid(const std::string& digits, int n_wall, int n_radial,
                          double far_field_radius);
Cloud load_cloud(const std::string& path);
void save_cloud(const Cloud& c, const std::string& path);
void save_cloud_binary(const Cloud& c, const std::string& path);  // load_cloud reads both formats
Cloud cloud_from_arrays(int n, const double* x, const double* y, const int* kind,
                        const double* nx, const double* ny, const int* off, const int* idx);

// classify + build_split_stencils + build_ls_coefficients + color_points.
void finalize(Cloud& c);

}  // namespace kfb
