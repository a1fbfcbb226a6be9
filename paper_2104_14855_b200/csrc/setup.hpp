// setup.hpp -- host-side setup stage of libmhdp: nested
// structured meshes, canonical numbering, free DoFs, vertex-star patches, operator
// assembly by rediscretisation and the exact FE prolongation.  Product code: it shares
// nothing with oracle/ (an independent implementation of the same definitions).
#pragma once
#include <cstdint>
#include <string>
#include <vector>

namespace mhdp {

struct Params {
    double Re = 1, Rem = 1, S = 1, gamma = 1, sigma = 10, mu = 0, theta = 1;
    int nu_pre = 1, nu_post = 1;
    int smoother = 0, smoother_its = 6;   // 0 Richardson sweeps, 1 GMRES(m) (NEXT-1)
    double dt = 0;                         // NEXT-4: > 0 -> transient, (1/dt) mass terms
    int picard = 0;                        // NEXT-4: 1 -> Picard, no G~ term
    int degree = 1;                        // NEXT-2: element degree k (2: 2D E-B, CG2 x RT2)
    int weights_mode = 0;                  // 0 by degree, 1 per-DoF 1/m_d, 2 uniform 1/max m_d
    int newton_reaction = 0;               // accepted; zero under R-w (reading R-newton)
};

// One level of the hierarchy as host arrays (the form both mhdp_assemble and
// mhdp_load_level produce).
struct HostLevel {
    int64_t n = 0;
    std::vector<int64_t> rp;   // CSR of A_l
    std::vector<int> ci;
    std::vector<double> v;
    std::vector<int64_t> pptr; // vertex-star patches, ascending DoFs
    std::vector<int> pdofs;
    std::vector<int> pvert;    // mesh vertex of each patch (mesh path; empty for mhdp_load_level)
    std::vector<int64_t> prp;  // prolongation from level-1 (rows: this level)
    std::vector<int> pci;
    std::vector<double> pv;
    int64_t n_coarser = 0;
};

// Assemble all levels (0 = coarsest).  block 0 = E-B, 1 = AL velocity.
// w: potential of the advecting field at the finest vertices (1 or 3 per vertex).
// Returns "" on success, else an error message.
// bn: potential of the magnetic field B^n (as w) for the Lorentz term of the velocity block
// (NEXT-4), or NULL
std::string assemble_hierarchy(int block, int dim, int N, int nlev, const Params &p, const double *w,
                               const double *bn, std::vector<HostLevel> &out);

// NEXT-3: the coupling blocks of the 4x4 Newton system (Table 1) on the finest
// mesh, as CSR (rows sorted), and the sizes of the four fields.
struct HostCsr {
    int64_t n = 0, ncols = 0;
    std::vector<int64_t> rp;
    std::vector<int> ci;
    std::vector<double> v;
};
struct CouplingBlocks {
    int64_t nu = 0, np = 0, nE = 0, nB = 0;
    HostCsr Bt;   // u x p   : -(q, div v)
    HostCsr J;    // u x E   : S (B^n x E, v)
    HostCsr Dt;   // u x B   : S (B x (u^n x B^n), v) + S (B^n x (u^n x B), v)   (0 under Picard)
    HostCsr G;    // E x u   : (u x B^n, F)
};
// floor_u[r] (r < nu) / floor_E[r] (r < nE): max |entry| of row r of the finest velocity /
// E-B matrix (fp64), or NULL: the coupling rows are rounded on the grid of the whole
// Newton row (reading R-cgrid of DESIGN.md).
std::string assemble_coupling(int dim, int N, const Params &p, const double *w, const double *bn, const double *floor_u,
                              const double *floor_E, CouplingBlocks &out);

}  // namespace mhdp
