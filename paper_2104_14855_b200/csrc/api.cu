// api.cu -- the C-ABI of include/mhdp.h: context, device stores, setup (K6/K7), the
// smoother and V-cycle drivers, GMRES and the export calls.
//
// Paper: arXiv 2104.14855.  Sweep = parallel subspace correction P:529-538; stars
// P:567-571; nested hierarchy + FE prolongation P:572; V-cycle with patch relaxation
// and a direct coarse solve P:643; right-preconditioned Krylov with the paper's
// 1e-7 tolerances P:625.  Readings (R-*) are listed in DESIGN.md.
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <chrono>
#include <cstring>
#include <string>
#include <vector>
#include <numeric>

#include "../../include/mhdp.h"
#include "kernels.cuh"
#include "setup.hpp"

#include <functional>

using namespace mhdp;

namespace {

struct DevLevel {
    int64_t n = 0, nnz = 0;
    DevSell A;
    DevBSell3 A3;
    bool use_b3 = false;
    DevPatches P;
    DevCsr Pr, PrT;            // prolongation from level-1 (fine rows) and its transpose
    double *b = nullptr, *x = nullptr, *r = nullptr;
    int64_t bytes_op = 0, bytes_fac = 0, bytes_tr = 0;
    // GMRES(m) smoother workspace (NEXT-1)
    double *gV = nullptr, *gt = nullptr, *gw = nullptr, *part = nullptr;
    double *scal = nullptr;    // H (m+1)m | cs m | sn m | g m+1 | y m | hn m
    int *kk = nullptr;         // device Krylov dimension (breakdown handling)
    int gm = 0;                // smoother iterations the workspace holds
};

}  // namespace

struct mhdp_ctx {
    int device = -1;
    cudaStream_t stream = nullptr;
    bool host_only = true;
    int nlev = 0;
    int block = -1;
    Params p;
    std::vector<HostLevel> H;
    std::vector<char> loaded;
    std::vector<DevLevel> D;
    bool setup_done = false;
    // coarse factor
    int n0 = 0;
    int *cperm = nullptr;      // R-lu row permutation of the coarse operator
    double *ctile = nullptr;   // K8 factor tiles of both substitution passes (k8_coarse.cu)
    double *crec = nullptr;    // K8 mini-block coefficient records
    double *czf = nullptr;     // forward-pass z (global copy for K8's far warps)
    double *chacc = nullptr;   // K8 far-warp partial sums
    double *cb = nullptr;      // copy of b when a caller aliases b and x
    unsigned long long *csync = nullptr;   // K8 epoch / progress / hand-off flags
    // scratch
    int *d_status = nullptr;
    double *d_scal = nullptr;  // dot partials + results
    std::vector<void *> allocs;
    std::string err;
    long long where = -1;
    long long launches0 = 0;
    double *vh = nullptr;      // mhdp_vcycle_host: device x of the finest level
    // setup timings (mhdp_setup_timings): device ms of K6 per level, K7, K8 pack; wall s
    std::vector<double> t_k6;
    double t_k7 = 0, t_k8pack = 0, t_setup_wall = 0;
    std::vector<double> t_stage;   // host wall s per setup stage (mhdp_setup_timings)
    // fgmres workspace
    double *fV = nullptr, *fZ = nullptr, *fw = nullptr, *fpart = nullptr, *fscal = nullptr;
    int f_cap = 0;
    // CUDA graphs of mhdp_vcycle, keyed by (level, b, x, smoother): the first call with a
    // key runs directly, the second captures the V-cycle on a private stream, later calls
    // replay it on the context stream
    struct VGraph {
        int level, smoother, its;
        const double *b;
        double *x;
        int calls = 0;
        cudaGraphExec_t exec = nullptr;
        long long nkern = 0;
    };
    std::vector<VGraph> graphs;
    cudaStream_t cap = nullptr;
    bool graphs_off = false;       // capture failed once: run uncaptured from then on
    bool graphs_disabled = false;  // mhdp_set_graphs(ctx, 0)
    // mhdp_vcycle_host_batch: two device (b, x) slots, copy-in / copy-out streams
    double *hb[2] = {nullptr, nullptr}, *hx[2] = {nullptr, nullptr};
    cudaStream_t s_in = nullptr, s_out = nullptr;
    cudaEvent_t ev_start = nullptr, ev_in[2] = {nullptr, nullptr}, ev_done[2] = {nullptr, nullptr},
                ev_out[2] = {nullptr, nullptr};
};

namespace {

mhdp_status fail(mhdp_ctx *c, mhdp_status st, const std::string &msg, long long where = -1) {
    if (c) { c->err = msg; c->where = where; }
    return st;
}

// scoped temporary device buffer (freed on every return path of the setup stages)
template <class T>
struct TmpDev {
    T *p = nullptr;
    ~TmpDev() { if (p) cudaFree(p); }
};

// CUDA-event stopwatch on a stream (setup diagnostics); stop() synchronises the event
struct EvTimer {
    cudaEvent_t a = nullptr, b = nullptr;
    cudaStream_t s;
    explicit EvTimer(cudaStream_t st) : s(st) {
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        cudaEventRecord(a, s);
    }
    double stop() {
        float ms = 0;
        cudaEventRecord(b, s);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        return ms;
    }
    ~EvTimer() {
        if (a) cudaEventDestroy(a);
        if (b) cudaEventDestroy(b);
    }
};

#define CK(call)                                                                              \
    do {                                                                                      \
        cudaError_t e_ = (call);                                                              \
        if (e_ != cudaSuccess)                                                                \
            return fail(ctx, MHDP_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
    } while (0)

// setup copies are stream-ordered on the context stream (which may be a non-blocking
// stream) and complete before returning, so pageable host buffers may be freed at once
cudaError_t h2d(const mhdp_ctx *ctx, void *dst, const void *src, size_t bytes) {
    cudaError_t e = cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, ctx->stream);
    return e != cudaSuccess ? e : cudaStreamSynchronize(ctx->stream);
}
cudaError_t d2h(const mhdp_ctx *ctx, void *dst, const void *src, size_t bytes) {
    cudaError_t e = cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, ctx->stream);
    return e != cudaSuccess ? e : cudaStreamSynchronize(ctx->stream);
}

template <class T>
mhdp_status dalloc(mhdp_ctx *ctx, T **p, int64_t count) {
    *p = nullptr;
    if (count <= 0) count = 1;
    cudaError_t e = cudaMalloc((void **)p, sizeof(T) * (size_t)count);
    if (e != cudaSuccess) {
        *p = nullptr;
        return fail(ctx, MHDP_ENOMEM, std::string("cudaMalloc: ") + cudaGetErrorString(e));
    }
    ctx->allocs.push_back(*p);
    return MHDP_OK;
}

template <class T>
mhdp_status upload(mhdp_ctx *ctx, T **p, const T *src, int64_t count) {
    mhdp_status st = dalloc(ctx, p, count);
    if (st) return st;
    if (count > 0) CK(h2d(ctx, *p, src, sizeof(T) * (size_t)count));
    return MHDP_OK;
}

mhdp_status check_launch(mhdp_ctx *ctx) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(ctx, MHDP_ECUDA, std::string("kernel launch: ") + cudaGetErrorString(e));
    return MHDP_OK;
}

void drop_graphs(mhdp_ctx *c) {
    for (auto &g : c->graphs)
        if (g.exec) cudaGraphExecDestroy(g.exec);
    c->graphs.clear();
}

void free_device(mhdp_ctx *c) {
    if (c->host_only) return;
    cudaSetDevice(c->device);
    cudaStreamSynchronize(c->stream);
    drop_graphs(c);
    for (void *p : c->allocs) cudaFree(p);
    c->allocs.clear();
    c->D.clear();
    c->cperm = nullptr; c->ctile = c->crec = c->czf = c->chacc = c->cb = nullptr; c->csync = nullptr;
    c->d_status = nullptr; c->d_scal = nullptr;
    c->fV = c->fZ = c->fw = c->fpart = c->fscal = nullptr; c->f_cap = 0;
    c->vh = nullptr;
    c->hb[0] = c->hb[1] = c->hx[0] = c->hx[1] = nullptr;
    c->setup_done = false;
}

bool valid_level(const mhdp_ctx *c, int l) { return c && l >= 0 && l < c->nlev; }

// ---------------- host -> device store construction ----------------

mhdp_status make_sell(mhdp_ctx *ctx, const HostLevel &H, DevSell &A, int64_t *bytes) {
    const int64_t n = H.n, ns = (n + 31) / 32;
    std::vector<int64_t> sptr(ns + 1, 0);
    std::vector<int> rlen(n);
    for (int64_t s = 0; s < ns; ++s) {
        int mx = 0;
        for (int64_t r = 32 * s; r < std::min(n, 32 * s + 32); ++r) {
            rlen[r] = (int)(H.rp[r + 1] - H.rp[r]);
            mx = std::max(mx, rlen[r]);
        }
        sptr[s + 1] = sptr[s] + 32 * (int64_t)mx;
    }
    const int64_t stored = sptr[ns];
    std::vector<int> col(stored, 0);
    std::vector<double> val(stored, 0.0);
#pragma omp parallel for schedule(static)
    for (int64_t r = 0; r < n; ++r) {
        const int64_t base = sptr[r >> 5] + (r & 31);
        for (int k = 0; k < rlen[r]; ++k) {
            col[base + 32 * k] = H.ci[H.rp[r] + k];
            val[base + 32 * k] = H.v[H.rp[r] + k];
        }
    }
    mhdp_status st;
    A.n = n; A.nslices = ns; A.stored = stored;
    if ((st = upload(ctx, &A.sptr, sptr.data(), ns + 1))) return st;
    if ((st = upload(ctx, &A.rlen, rlen.data(), n))) return st;
    if ((st = upload(ctx, &A.col, col.data(), stored))) return st;
    if ((st = upload(ctx, &A.val, val.data(), stored))) return st;
    if (bytes) *bytes = 8 * (ns + 1) + 4 * n + 12 * stored;
    return MHDP_OK;
}

mhdp_status build_sell(mhdp_ctx *ctx, const HostLevel &H, DevLevel &L) { return make_sell(ctx, H, L.A, &L.bytes_op); }


// aligned 3x3 block structure: n % 3 == 0, rows 3R..3R+2 share one column list made of
// complete aligned triples
bool has_block3(const HostLevel &H) {
    if (H.n == 0 || H.n % 3) return false;
    bool ok = true;
#pragma omp parallel for schedule(static) reduction(&& : ok)
    for (int64_t R = 0; R < H.n / 3; ++R) {
        const int64_t a = H.rp[3 * R], len = H.rp[3 * R + 1] - a;
        bool r_ok = len % 3 == 0;
        for (int q = 1; q < 3 && r_ok; ++q) {
            if (H.rp[3 * R + q + 1] - H.rp[3 * R + q] != len) r_ok = false;
            else if (!std::equal(H.ci.begin() + a, H.ci.begin() + a + len, H.ci.begin() + H.rp[3 * R + q])) r_ok = false;
        }
        for (int64_t t = 0; t < len && r_ok; t += 3) {
            const int c = H.ci[a + t];
            if (c % 3 || H.ci[a + t + 1] != c + 1 || H.ci[a + t + 2] != c + 2) r_ok = false;
        }
        ok = ok && r_ok;
    }
    return ok;
}

// The 3x3-block SELL store is filled on the device from the level's CSR (drp / dci / dv, the
// temporary copy K6 factors from): only the slice pointers and row lengths are formed on the
// host.  (Round 1 filled 2.4 GB of values on the host and uploaded them from pageable memory:
// 1.4 s of the c5 device setup.)
mhdp_status build_b3(mhdp_ctx *ctx, const HostLevel &H, DevLevel &L, const int64_t *drp, const int *dci,
                     const double *dv) {
    const int64_t nb = H.n / 3, ns = (nb + 31) / 32;
    std::vector<int64_t> sptr(ns + 1, 0);
    std::vector<int> rlen(nb);
    for (int64_t s = 0; s < ns; ++s) {
        int mx = 0;
        for (int64_t R = 32 * s; R < std::min(nb, 32 * s + 32); ++R) {
            rlen[R] = (int)((H.rp[3 * R + 1] - H.rp[3 * R]) / 3);
            mx = std::max(mx, rlen[R]);
        }
        sptr[s + 1] = sptr[s] + 32 * (int64_t)mx;
    }
    const int64_t stored = sptr[ns];
    // value layout: the 9 x 32 values of one (slice, block column) contiguous (one DRAM run
    // per warp iteration; 9 separate planes measured 3% slower, profiles/r01_c5_k1_layout_ab.jsonl)
    mhdp_status st;
    L.A3.nb = nb; L.A3.nslices = ns; L.A3.stored = stored; L.A3.planes = 0;
    if ((st = upload(ctx, &L.A3.sptr, sptr.data(), ns + 1))) return st;
    if ((st = upload(ctx, &L.A3.rlen, rlen.data(), nb))) return st;
    if ((st = dalloc(ctx, &L.A3.col, stored))) return st;
    if ((st = dalloc(ctx, &L.A3.val, 9 * stored))) return st;
    CK(cudaMemsetAsync(L.A3.col, 0, sizeof(int) * (size_t)std::max<int64_t>(1, stored), ctx->stream));
    CK(cudaMemsetAsync(L.A3.val, 0, sizeof(double) * (size_t)std::max<int64_t>(1, 9 * stored), ctx->stream));
    launch_build_b3(L.A3, drp, dci, dv, ctx->stream);
    if ((st = check_launch(ctx))) return st;
    L.bytes_op = 8 * (ns + 1) + 4 * nb + 76 * stored;
    return MHDP_OK;
}

mhdp_status build_csr(mhdp_ctx *ctx, int64_t n, const std::vector<int64_t> &rp, const std::vector<int> &ci,
                      const std::vector<double> &v, DevCsr &out) {
    std::vector<int> rp32(n + 1);
    for (int64_t i = 0; i <= n; ++i) rp32[i] = (int)rp[i];
    out.n = n; out.nnz = rp[n];
    mhdp_status st;
    if ((st = upload(ctx, &out.rp, rp32.data(), n + 1))) return st;
    if ((st = upload(ctx, &out.ci, ci.data(), out.nnz))) return st;
    if ((st = upload(ctx, &out.v, v.data(), out.nnz))) return st;
    return MHDP_OK;
}

void transpose_csr(int64_t n, int64_t ncols, const std::vector<int64_t> &rp, const std::vector<int> &ci,
                   const std::vector<double> &v, std::vector<int64_t> &trp, std::vector<int> &tci,
                   std::vector<double> &tv) {
    trp.assign(ncols + 1, 0);
    for (int64_t t = 0; t < rp[n]; ++t) trp[ci[t] + 1]++;
    for (int64_t j = 0; j < ncols; ++j) trp[j + 1] += trp[j];
    tci.resize(rp[n]);
    tv.resize(rp[n]);
    std::vector<int64_t> pos(trp.begin(), trp.end() - 1);
    for (int64_t i = 0; i < n; ++i)       // ascending fine rows => each coarse row ascending
        for (int64_t t = rp[i]; t < rp[i + 1]; ++t) {
            const int64_t q = pos[ci[t]]++;
            tci[q] = (int)i;
            tv[q] = v[t];
        }
}

mhdp_status build_patches(mhdp_ctx *ctx, const HostLevel &H, DevLevel &L) {
    DevPatches &P = L.P;
    const int64_t np = (int64_t)H.pptr.size() - 1, sum_n = H.pptr[np];
    P.np = np; P.sum_n = sum_n;
    std::vector<int> pn(np);
    std::vector<int64_t> foff(np);
    int64_t f = 0;
    int mx = 0;
    for (int64_t i = 0; i < np; ++i) {
        pn[i] = (int)(H.pptr[i + 1] - H.pptr[i]);
        mx = std::max(mx, pn[i]);
        foff[i] = f;
        f += ((int64_t)pn[i] * pn[i] + pn[i] + 15) / 16 * 16;   // packed stream n^2+n, 128-byte aligned
    }
    if (mx > K2_MAX_N) return fail(ctx, MHDP_EINVAL, "patch larger than 384 DoFs is not supported");
    P.max_n = mx;
    P.fac_doubles = f;
    std::vector<int> mult(H.n, 0);
    for (int64_t t = 0; t < sum_n; ++t) mult[H.pdofs[t]]++;
    std::vector<int> dptr(H.n + 1, 0);
    for (int64_t d = 0; d < H.n; ++d) {
        if (mult[d] == 0) return fail(ctx, MHDP_EINVAL, "a DoF is covered by no patch", d);
        dptr[d + 1] = dptr[d] + mult[d];
    }
    std::vector<int> dslot(sum_n), fill(dptr.begin(), dptr.end() - 1);
    for (int64_t t = 0; t < sum_n; ++t) dslot[fill[H.pdofs[t]]++] = (int)t;   // ascending slot = ascending patch
    // R-weights (k = 1): theta / m_d;  R-weights2 (k = 2): the uniform theta / max_d m_d (a
    // per-subspace damping parameter of P:538 that keeps local kernel corrections in the kernel)
    // weights_mode: 1 per-DoF, 2 uniform, 0 by degree
    const bool uniform = ctx->p.weights_mode == 2 || (ctx->p.weights_mode == 0 && ctx->p.degree == 2);
    int mmax = 1;
    for (int64_t d = 0; d < H.n; ++d) mmax = std::max(mmax, mult[d]);
    std::vector<double> wd(H.n);
    for (int64_t d = 0; d < H.n; ++d)
        wd[d] = ctx->p.theta * (1.0 / (uniform ? mmax : mult[d]));
    mhdp_status st;
    if ((st = upload(ctx, &P.pn, pn.data(), np))) return st;
    if ((st = upload(ctx, &P.poff, H.pptr.data(), np))) return st;
    if ((st = upload(ctx, &P.foff, foff.data(), np))) return st;
    {   // walk order of the persistent K2 kernels: size descending, stable
        std::vector<int64_t> ord(np);
        std::iota(ord.begin(), ord.end(), 0);
        std::stable_sort(ord.begin(), ord.end(), [&](int64_t a, int64_t b) { return pn[a] > pn[b]; });
        std::vector<int> pno(np);
        std::vector<int64_t> poo(np), foo(np);
        for (int64_t k = 0; k < np; ++k) { pno[k] = pn[ord[k]]; poo[k] = H.pptr[ord[k]]; foo[k] = foff[ord[k]]; }
        if ((st = upload(ctx, &P.pn_o, pno.data(), np))) return st;
        if ((st = upload(ctx, &P.poff_o, poo.data(), np))) return st;
        if ((st = upload(ctx, &P.foff_o, foo.data(), np))) return st;
    }
    if ((st = upload(ctx, &P.pdofs, H.pdofs.data(), sum_n))) return st;
    if ((st = dalloc(ctx, &P.gidx, sum_n))) return st;
    if ((st = dalloc(ctx, &P.perm, sum_n))) return st;
    if ((st = dalloc(ctx, &P.fac, f))) return st;
    if ((st = upload(ctx, &P.dptr, dptr.data(), H.n + 1))) return st;
    if ((st = upload(ctx, &P.dslot, dslot.data(), sum_n))) return st;
    // DoF triples (3D velocity: the 3 DoFs of a face) whose slot lists are the same patches
    // at consecutive slots: K3 can update a triple per thread from one slot list
    P.triples = H.n % 3 == 0 && H.n > 0;
    for (int64_t R = 0; P.triples && R < H.n / 3; ++R) {
        const int64_t d = 3 * R;
        const int m = dptr[d + 1] - dptr[d];
        if (dptr[d + 2] - dptr[d + 1] != m || dptr[d + 3] - dptr[d + 2] != m) { P.triples = false; break; }
        for (int k = 0; k < m; ++k)
            if (dslot[dptr[d + 1] + k] != dslot[dptr[d] + k] + 1 || dslot[dptr[d + 2] + k] != dslot[dptr[d] + k] + 2) {
                P.triples = false;
                break;
            }
    }
    if ((st = upload(ctx, &P.wd, wd.data(), H.n))) return st;
    if ((st = dalloc(ctx, &P.y, sum_n))) return st;
    L.bytes_fac = 8 * f + 4 * np + 16 * np + 12 * sum_n;
    return MHDP_OK;
}

// small stars: group the patches 32 at a time by size and interleave their factor streams
// (K2 thread-per-patch kernel)
mhdp_status build_lane_groups(mhdp_ctx *ctx, const HostLevel &H, DevLevel &L) {
    DevPatches &P = L.P;
    // measured (tools/level_profile.py, profiles/r01_k2_lring_ab.jsonl): the ring-fed
    // thread-per-patch kernel wins wherever the level has enough 32-patch groups to keep
    // every warp busy (a group of 31/36-DoF stars is a ~40-50 us chain per thread), or
    // the stars are small: k = 2 E-B finest 5.7 vs 2.8 TB/s, c3 finest 4.6 vs 2.0 TB/s
    if (P.np == 0) return MHDP_OK;
    if (!(P.max_n <= 16 || P.np >= 40000)) return MHDP_OK;
    for (int64_t i = 0; i < P.np; ++i)
        if (!lring_size_supported((int)(H.pptr[i + 1] - H.pptr[i]))) return MHDP_OK;
    const int64_t np = P.np;
    std::vector<int64_t> order(np);
    std::iota(order.begin(), order.end(), 0);
    auto sz = [&](int64_t i) { return (int)(H.pptr[i + 1] - H.pptr[i]); };
    std::stable_sort(order.begin(), order.end(), [&](int64_t a, int64_t b) { return sz(a) < sz(b); });
    std::vector<int> gn, gpatch;
    std::vector<int64_t> gbase;
    int64_t tot = 0;
    for (int64_t k = 0; k < np;) {
        const int n = sz(order[k]);
        int64_t k1 = k;
        while (k1 < np && k1 - k < 32 && sz(order[k1]) == n) ++k1;
        gn.push_back(n);
        gbase.push_back(tot);
        for (int t = 0; t < 32; ++t) gpatch.push_back(k + t < k1 ? (int)order[k + t] : -1);
        tot += 32 * ((int64_t)n * n + n);
        k = k1;
    }
    P.ng = (int64_t)gn.size();
    mhdp_status st;
    if ((st = upload(ctx, &P.gn, gn.data(), P.ng))) return st;
    if ((st = upload(ctx, &P.gbase, gbase.data(), P.ng))) return st;
    if ((st = upload(ctx, &P.gpatch, gpatch.data(), 32 * P.ng))) return st;
    if ((st = dalloc(ctx, &P.facI, tot))) return st;
    launch_interleave(P, ctx->stream);
    if ((st = check_launch(ctx))) return st;
    CK(cudaStreamSynchronize(ctx->stream));
    L.bytes_fac += 8 * tot;
    return MHDP_OK;
}

// ---------------- device drivers ----------------

void residual(mhdp_ctx *ctx, int l, const double *b, const double *x, double *r) {
    DevLevel &L = ctx->D[l];
    if (L.use_b3) launch_residual_b3(L.A3, b, x, r, ctx->stream);
    else launch_residual(L.A, b, x, r, ctx->stream);
}

void sweep(mhdp_ctx *ctx, int l, const double *b, double *x, bool x_zero) {
    DevLevel &L = ctx->D[l];
    const double *r = b;
    if (!x_zero) {
        residual(ctx, l, b, x, L.r);
        r = L.r;
    }
    launch_patch_apply(L.P, r, ctx->stream);
    launch_patch_update(L.P, L.n, x, x_zero ? 1 : 0, ctx->stream);
}

void coarse_solve(mhdp_ctx *ctx, const double *b, double *x) {
    if (b == x) {   // K8 reads b while it writes x
        cudaMemcpyAsync(ctx->cb, b, sizeof(double) * ctx->n0, cudaMemcpyDeviceToDevice, ctx->stream);
        b = ctx->cb;
    }
    launch_k8_solve(ctx->ctile, ctx->crec, ctx->cperm, ctx->n0, b, x, ctx->czf, ctx->chacc, ctx->csync,
                    ctx->stream);
}

// scalar workspace layout of a GMRES(m) smoother / FGMRES(m)
struct KrylovScal {
    double *H, *cs, *sn, *g, *y, *hn;
    KrylovScal(double *s, int m) {
        H = s; cs = H + (m + 1) * m; sn = cs + m; g = sn + m; y = g + m + 1; hn = y + m;
    }
    static int64_t size(int m) { return (int64_t)(m + 1) * m + 5 * (int64_t)m + 1; }
};

// NEXT-1 smoothing step (R-gmres6): left-preconditioned GMRES(m) from the current x
// (x_is_zero: x = 0 on entry), preconditioner B r = one Schwarz sweep from zero.
void gmres_smooth(mhdp_ctx *ctx, int l, int m, bool x_is_zero, const double *b, double *x) {
    DevLevel &L = ctx->D[l];
    cudaStream_t s = ctx->stream;
    const int64_t n = L.n;
    KrylovScal S(L.scal, m);
    auto applyB = [&](const double *rhs, double *out) {
        launch_patch_apply(L.P, rhs, s);
        launch_patch_update(L.P, n, out, 1, s);
    };
    const double *r = b;
    if (x_is_zero) launch_fill(x, 0.0, n, s);
    else { residual(ctx, l, b, x, L.r); r = L.r; }
    applyB(r, L.gw);
    launch_dot_pinned(L.gw, L.gw, n, L.part, S.g, 1, s);                  // beta -> g[0]
    launch_krylov_init(S.g, m, L.kk, s);                                  // kk = 0 if beta == 0
    launch_div_dev(L.gV, L.gw, S.g, n, s);                                // V_0 = w / beta
    for (int k = 0; k < m; ++k) {
        residual(ctx, l, nullptr, L.gV + (int64_t)k * n, L.gt);           // t = A V_k
        applyB(L.gt, L.gw);                                               // w = B t
        for (int i = 0; i <= k; ++i) {
            launch_dot_pinned(L.gw, L.gV + (int64_t)i * n, n, L.part, S.H + i * m + k, 0, s);
            launch_axpy_negdev(L.gw, S.H + i * m + k, L.gV + (int64_t)i * n, n, s);
        }
        launch_dot_pinned(L.gw, L.gw, n, L.part, S.hn + k, 1, s);
        launch_givens(S.H, m, S.cs, S.sn, S.g, S.hn + k, k, L.kk, s);
        if (k + 1 < m) launch_div_dev(L.gV + (int64_t)(k + 1) * n, L.gw, S.hn + k, n, s);
    }
    launch_backsub(S.H, m, S.g, m, L.kk, S.y, s);          // uses the device kk (<= m)
    launch_basis_update(x, L.gV, n, S.y, m, L.kk, n, s);
}

// GMRES(m) smoother workspace of one level (allocated at setup or by mhdp_set_smoother)
mhdp_status alloc_smoother(mhdp_ctx *ctx, DevLevel &L, int m) {
    mhdp_status st;
    if (L.gm >= m) return MHDP_OK;
    if ((st = dalloc(ctx, &L.gV, (int64_t)(m + 1) * L.n))) return st;
    if (!L.gt && (st = dalloc(ctx, &L.gt, L.n))) return st;
    if (!L.gw && (st = dalloc(ctx, &L.gw, L.n))) return st;
    if (!L.part && (st = dalloc(ctx, &L.part, 2 * ((L.n + 255) / 256) + 2))) return st;
    if ((st = dalloc(ctx, &L.scal, KrylovScal::size(m)))) return st;
    if (!L.kk && (st = dalloc(ctx, &L.kk, 1))) return st;
    L.gm = m;
    return MHDP_OK;
}

void vcycle(mhdp_ctx *ctx, int l, const double *b, double *x) {
    if (l == 0) {
        coarse_solve(ctx, b, x);
        return;
    }
    DevLevel &L = ctx->D[l];
    DevLevel &C = ctx->D[l - 1];
    const bool krylov = ctx->p.smoother == 1;
    if (krylov) gmres_smooth(ctx, l, ctx->p.smoother_its, true, b, x);
    else {
        if (ctx->p.nu_pre == 0) launch_fill(x, 0.0, L.n, ctx->stream);
        for (int s = 0; s < ctx->p.nu_pre; ++s) sweep(ctx, l, b, x, s == 0);
    }
    residual(ctx, l, b, x, L.r);
    launch_restrict(L.PrT, L.r, C.b, ctx->stream);
    vcycle(ctx, l - 1, C.b, C.x);
    launch_prolong_add(L.Pr, C.x, x, ctx->stream);
    if (krylov) gmres_smooth(ctx, l, ctx->p.smoother_its, false, b, x);
    else
        for (int s = 0; s < ctx->p.nu_post; ++s) sweep(ctx, l, b, x, false);
}

mhdp_status need_setup(mhdp_ctx *ctx) {
    if (!ctx) return MHDP_EINVAL;
    if (ctx->host_only) return fail(ctx, MHDP_ECUDA, "host-only context (created with cuda_device = -1)");
    if (!ctx->setup_done) return fail(ctx, MHDP_ESTATE, "mhdp_setup has not completed");
    cudaSetDevice(ctx->device);
    return MHDP_OK;
}

mhdp_status validate_level(mhdp_ctx *ctx, const HostLevel &H, int level) {
    if (H.n < 0 || (int64_t)H.rp.size() != H.n + 1 || H.rp[0] != 0) return fail(ctx, MHDP_EINVAL, "bad row pointer");
    for (int64_t i = 0; i < H.n; ++i) {
        if (H.rp[i + 1] < H.rp[i]) return fail(ctx, MHDP_EINVAL, "row pointer not monotone", i);
        for (int64_t t = H.rp[i]; t < H.rp[i + 1]; ++t) {
            if (H.ci[t] < 0 || H.ci[t] >= H.n) return fail(ctx, MHDP_EINVAL, "column out of range", i);
            if (t > H.rp[i] && H.ci[t] <= H.ci[t - 1]) return fail(ctx, MHDP_EINVAL, "columns not ascending", i);
        }
    }
    if (level > 0) {
        const int64_t np = (int64_t)H.pptr.size() - 1;
        if (np < 0 || H.pptr[0] != 0) return fail(ctx, MHDP_EINVAL, "bad patch pointer");
        for (int64_t i = 0; i < np; ++i) {
            if (H.pptr[i + 1] <= H.pptr[i]) return fail(ctx, MHDP_EINVAL, "empty patch", i);
            for (int64_t t = H.pptr[i]; t < H.pptr[i + 1]; ++t) {
                if (H.pdofs[t] < 0 || H.pdofs[t] >= H.n) return fail(ctx, MHDP_EINVAL, "patch DoF out of range", i);
                if (t > H.pptr[i] && H.pdofs[t] <= H.pdofs[t - 1])
                    return fail(ctx, MHDP_EINVAL, "patch DoFs not ascending", i);
            }
        }
        if ((int64_t)H.prp.size() != H.n + 1) return fail(ctx, MHDP_EINVAL, "bad prolongation row pointer");
        for (int64_t t = 0; t < H.prp[H.n]; ++t)
            if (H.pci[t] < 0 || H.pci[t] >= H.n_coarser) return fail(ctx, MHDP_EINVAL, "prolongation column out of range");
    }
    return MHDP_OK;
}

}  // namespace

// =====================================================================================
extern "C" {

mhdp_status mhdp_create(mhdp_ctx **out, int cuda_device, void *cuda_stream) {
    if (!out) return MHDP_EINVAL;
    *out = nullptr;
    mhdp_ctx *ctx = new (std::nothrow) mhdp_ctx();
    if (!ctx) return MHDP_ENOMEM;
    if (cuda_device >= 0) {
        int cnt = 0;
        if (cudaGetDeviceCount(&cnt) != cudaSuccess || cuda_device >= cnt) {
            delete ctx;
            return MHDP_ECUDA;
        }
        if (cudaSetDevice(cuda_device) != cudaSuccess) { delete ctx; return MHDP_ECUDA; }
        ctx->device = cuda_device;
        ctx->host_only = false;
        ctx->stream = (cudaStream_t)cuda_stream;
        ctx->launches0 = g_launches;
    }
    *out = ctx;
    return MHDP_OK;
}

void mhdp_destroy(mhdp_ctx *ctx) {
    if (!ctx) return;
    free_device(ctx);
    if (ctx->cap) cudaStreamDestroy(ctx->cap);
    if (ctx->s_in) cudaStreamDestroy(ctx->s_in);
    if (ctx->s_out) cudaStreamDestroy(ctx->s_out);
    for (cudaEvent_t e : {ctx->ev_start, ctx->ev_in[0], ctx->ev_in[1], ctx->ev_done[0], ctx->ev_done[1], ctx->ev_out[0],
                          ctx->ev_out[1]})
        if (e) cudaEventDestroy(e);
    delete ctx;
}

static mhdp_status check_params(mhdp_ctx *ctx, const mhdp_params *pr) {
    if (!pr) return fail(ctx, MHDP_EINVAL, "params is NULL");
    if (!(pr->Re > 0) || !(pr->Rem > 0) || !(pr->gamma > 0) || !(pr->sigma > 0))
        return fail(ctx, MHDP_EINVAL, "Re, Rem, gamma and sigma must be positive");
    if (!(pr->mu_stab >= 0.0)) return fail(ctx, MHDP_EINVAL, "mu_stab must be >= 0");
    if (pr->mu_stab != 0.0 && pr->degree == 2)
        return fail(ctx, MHDP_EINVAL, "mu_stab > 0 is assembled for k = 1 only (reading R-mu)");
    if (pr->nu_pre < 0 || pr->nu_post < 0) return fail(ctx, MHDP_EINVAL, "negative sweep counts");
    if (!(pr->theta > 0)) return fail(ctx, MHDP_EINVAL, "theta must be positive");
    ctx->p.Re = pr->Re; ctx->p.Rem = pr->Rem; ctx->p.S = pr->S; ctx->p.gamma = pr->gamma;
    ctx->p.sigma = pr->sigma; ctx->p.mu = pr->mu_stab; ctx->p.theta = pr->theta;
    ctx->p.nu_pre = pr->nu_pre; ctx->p.nu_post = pr->nu_post;
    if (pr->smoother != 0 && pr->smoother != 1) return fail(ctx, MHDP_EINVAL, "smoother must be 0 or 1");
    if (pr->smoother == 1 && (pr->smoother_its < 1 || pr->smoother_its > 32))
        return fail(ctx, MHDP_EINVAL, "smoother_its must be in 1..32");
    ctx->p.smoother = pr->smoother; ctx->p.smoother_its = pr->smoother_its;
    if (pr->dt < 0 || pr->dt != pr->dt) return fail(ctx, MHDP_EINVAL, "dt must be >= 0");
    if (pr->picard != 0 && pr->picard != 1) return fail(ctx, MHDP_EINVAL, "picard must be 0 or 1");
    ctx->p.dt = pr->dt; ctx->p.picard = pr->picard;
    if (pr->degree < 0 || pr->degree > 2) return fail(ctx, MHDP_EINVAL, "degree must be 1 or 2");
    ctx->p.degree = pr->degree == 0 ? 1 : pr->degree;
    if (pr->weights_mode < 0 || pr->weights_mode > 2) return fail(ctx, MHDP_EINVAL, "weights_mode must be 0, 1 or 2");
    if (pr->newton_reaction != 0 && pr->newton_reaction != 1)
        return fail(ctx, MHDP_EINVAL, "newton_reaction must be 0 or 1");
    ctx->p.weights_mode = pr->weights_mode;
    ctx->p.newton_reaction = pr->newton_reaction;   // zero cellwise under R-w (reading R-newton)
    return MHDP_OK;
}

mhdp_status mhdp_assemble_lorentz(mhdp_ctx *ctx, mhdp_block block, const mhdp_mesh *mesh,
                                  const mhdp_params *params, const double *w_vertex_host,
                                  const double *bn_vertex_host) {
    if (!ctx) return MHDP_EINVAL;
    if (!mesh || !w_vertex_host) return fail(ctx, MHDP_EINVAL, "NULL mesh or w_vertex");
    if (block != MHDP_BLOCK_EB && block != MHDP_BLOCK_ALVEL) return fail(ctx, MHDP_EINVAL, "unknown block");
    if ((mesh->dim != 2 && mesh->dim != 3) || mesh->n_fine < 1 || mesh->n_levels < 1 || mesh->n_levels > 12)
        return fail(ctx, MHDP_EINVAL, "bad mesh dimensions");
    if (mesh->n_fine % (1 << (mesh->n_levels - 1)))
        return fail(ctx, MHDP_EINVAL, "n_fine must be divisible by 2^(n_levels-1)");
    mhdp_status st = check_params(ctx, params);
    if (st) return st;
    free_device(ctx);
    ctx->H.clear();
    if (bn_vertex_host && block != MHDP_BLOCK_ALVEL)
        return fail(ctx, MHDP_EINVAL, "the Lorentz term belongs to the velocity block");
    std::string e = assemble_hierarchy((int)block, mesh->dim, mesh->n_fine, mesh->n_levels, ctx->p, w_vertex_host,
                                       bn_vertex_host, ctx->H);
    if (!e.empty()) { ctx->H.clear(); ctx->nlev = 0; return fail(ctx, MHDP_EINVAL, e); }
    ctx->nlev = mesh->n_levels;
    ctx->block = (int)block;
    ctx->loaded.assign(ctx->nlev, 1);
    return MHDP_OK;
}

mhdp_status mhdp_assemble(mhdp_ctx *ctx, mhdp_block block, const mhdp_mesh *mesh, const mhdp_params *params,
                          const double *w_vertex_host) {
    return mhdp_assemble_lorentz(ctx, block, mesh, params, w_vertex_host, nullptr);
}

mhdp_status mhdp_begin_levels(mhdp_ctx *ctx, int n_levels, const mhdp_params *params) {
    if (!ctx) return MHDP_EINVAL;
    if (n_levels < 1 || n_levels > 16) return fail(ctx, MHDP_EINVAL, "bad n_levels");
    mhdp_status st = check_params(ctx, params);
    if (st) return st;
    free_device(ctx);
    ctx->H.assign(n_levels, HostLevel());
    ctx->loaded.assign(n_levels, 0);
    ctx->nlev = n_levels;
    ctx->block = -1;
    return MHDP_OK;
}

mhdp_status mhdp_load_level(mhdp_ctx *ctx, int level, long long n, const long long *rowptr, const int *col,
                            const double *val, long long npatch, const long long *pptr, const int *pdofs,
                            const long long *prow, const int *pcol, const double *pval) {
    if (!ctx) return MHDP_EINVAL;
    if (!valid_level(ctx, level) || (int)ctx->loaded.size() != ctx->nlev)
        return fail(ctx, MHDP_ESTATE, "mhdp_begin_levels first / bad level");
    if (n < 0 || !rowptr || (n > 0 && (!col || !val))) return fail(ctx, MHDP_EINVAL, "NULL operator arrays");
    if (level > 0 && (npatch < 1 || !pptr || !pdofs || !prow || !pcol || !pval))
        return fail(ctx, MHDP_EINVAL, "levels >= 1 need patches and a prolongation");
    if (level > 0 && !ctx->loaded[level - 1]) return fail(ctx, MHDP_ESTATE, "load level-1 first");
    HostLevel H;
    H.n = n;
    H.rp.assign(rowptr, rowptr + n + 1);
    const int64_t nnz = H.rp[n];
    if (nnz < 0) return fail(ctx, MHDP_EINVAL, "bad row pointer");
    H.ci.assign(col, col + nnz);
    H.v.assign(val, val + nnz);
    if (level > 0) {
        H.pptr.assign(pptr, pptr + npatch + 1);
        H.pdofs.assign(pdofs, pdofs + H.pptr[npatch]);
        H.prp.assign(prow, prow + n + 1);
        H.pci.assign(pcol, pcol + H.prp[n]);
        H.pv.assign(pval, pval + H.prp[n]);
        H.n_coarser = ctx->H[level - 1].n;
    }
    mhdp_status st = validate_level(ctx, H, level);
    if (st) return st;
    free_device(ctx);
    ctx->H[level] = std::move(H);
    ctx->loaded[level] = 1;
    return MHDP_OK;
}

mhdp_status mhdp_setup(mhdp_ctx *ctx) {
    if (!ctx) return MHDP_EINVAL;
    if (ctx->host_only) return fail(ctx, MHDP_ECUDA, "host-only context (created with cuda_device = -1)");
    if (ctx->nlev < 1) return fail(ctx, MHDP_ESTATE, "nothing assembled");
    for (int l = 0; l < ctx->nlev; ++l)
        if (!ctx->loaded[l]) return fail(ctx, MHDP_ESTATE, "level not loaded", l);
    free_device(ctx);
    CK(cudaSetDevice(ctx->device));
    const auto wall0 = std::chrono::steady_clock::now();
    ctx->t_k6.assign(ctx->nlev, 0.0);
    ctx->t_stage.assign(6, 0.0);   // operator stores (+ CSR upload), patch stores, transfers, K6, lane groups, coarse
    auto tick = [last = std::chrono::steady_clock::now()](double &acc) mutable {
        const auto now = std::chrono::steady_clock::now();
        acc += std::chrono::duration<double>(now - last).count();
        last = now;
    };
    mhdp_status st;
    if ((st = dalloc(ctx, &ctx->d_status, 4))) return st;
    if ((st = dalloc(ctx, &ctx->d_scal, 2048))) return st;
    ctx->D.assign(ctx->nlev, DevLevel());
    for (int l = 0; l < ctx->nlev; ++l) {
        const HostLevel &H = ctx->H[l];
        DevLevel &L = ctx->D[l];
        L.n = H.n;
        L.nnz = H.rp[H.n];
        L.use_b3 = l > 0 && has_block3(H);
        // temporary device CSR of the level: the block store is filled from it and K6 factors from it
        TmpDev<int64_t> buf_rp;
        TmpDev<int> buf_ci;
        TmpDev<double> buf_v;
        if (l > 0) {
            CK(cudaMalloc(&buf_rp.p, sizeof(int64_t) * (H.n + 1)));
            CK(cudaMalloc(&buf_ci.p, sizeof(int) * std::max<int64_t>(1, L.nnz)));
            CK(cudaMalloc(&buf_v.p, sizeof(double) * std::max<int64_t>(1, L.nnz)));
            CK(h2d(ctx, buf_rp.p, H.rp.data(), sizeof(int64_t) * (H.n + 1)));
            CK(h2d(ctx, buf_ci.p, H.ci.data(), sizeof(int) * L.nnz));
            CK(h2d(ctx, buf_v.p, H.v.data(), sizeof(double) * L.nnz));
        }
        if ((st = L.use_b3 ? build_b3(ctx, H, L, buf_rp.p, buf_ci.p, buf_v.p) : build_sell(ctx, H, L))) return st;
        tick(ctx->t_stage[0]);
        if ((st = dalloc(ctx, &L.b, H.n))) return st;
        if ((st = dalloc(ctx, &L.x, H.n))) return st;
        if ((st = dalloc(ctx, &L.r, H.n))) return st;
        if (l == 0) continue;
        tick(ctx->t_stage[0]);
        if ((st = build_patches(ctx, H, L))) return st;
        tick(ctx->t_stage[1]);
        if (ctx->p.smoother == 1 && (st = alloc_smoother(ctx, L, ctx->p.smoother_its))) return st;
        if ((st = build_csr(ctx, H.n, H.prp, H.pci, H.pv, L.Pr))) return st;
        std::vector<int64_t> trp; std::vector<int> tci; std::vector<double> tv;
        transpose_csr(H.n, H.n_coarser, H.prp, H.pci, H.pv, trp, tci, tv);
        if ((st = build_csr(ctx, H.n_coarser, trp, tci, tv, L.PrT))) return st;
        L.bytes_tr = 2 * (12 * (int64_t)H.prp[H.n]) + 4 * (H.n + H.n_coarser + 2);
        tick(ctx->t_stage[2]);
        // K6: batched patch LU from the temporary device CSR
        int64_t *drp = buf_rp.p;
        int *dci = buf_ci.p;
        double *dv = buf_v.p;
        int big = INT_MAX;
        CK(h2d(ctx, ctx->d_status, &big, sizeof(int)));
        TmpDev<double> buf_lu;            // K6 scratch for stars beyond shared memory
        const int64_t nscr = patch_lu_scratch_doubles(L.P);
        if (nscr) CK(cudaMalloc(&buf_lu.p, sizeof(double) * nscr));
        EvTimer tk6(ctx->stream);
        launch_patch_lu(L.P, drp, dci, dv, ctx->d_status, buf_lu.p, ctx->stream);
        ctx->t_k6[l] = tk6.stop();
        if ((st = check_launch(ctx))) return st;
        CK(cudaStreamSynchronize(ctx->stream));
        int bad = 0;
        CK(d2h(ctx, &bad, ctx->d_status, sizeof(int)));
        if (bad != INT_MAX) {
            const long long patch = bad - 1;
            char buf[160];
            // ESINGULAR names the vertex whose star is singular (mesh path);
            // for operators installed by mhdp_load_level the patch index stands in for it
            const bool have_v = (int64_t)H.pvert.size() > patch;
            const long long vid = have_v ? H.pvert[patch] : patch;
            snprintf(buf, sizeof buf, "singular patch %lld (%s %lld) on level %d", patch,
                     have_v ? "vertex" : "patch", vid, l);
            return fail(ctx, MHDP_ESINGULAR, buf, vid);
        }
        tick(ctx->t_stage[3]);
        if ((st = build_lane_groups(ctx, H, L))) return st;
        tick(ctx->t_stage[4]);
    }
    // K7: coarse LU (dense, row-major, R-lu), then the K8 tiles of both substitution passes
    const HostLevel &H0 = ctx->H[0];
    const int64_t n0 = H0.n;
    if (n0 > std::min(k8_max_n(), k7_max_n())) return fail(ctx, MHDP_EINVAL, "coarse level too large for the dense LU");
    ctx->n0 = (int)n0;
    {
        std::vector<double> dense((size_t)(n0 * n0), 0.0);
        for (int64_t i = 0; i < n0; ++i)
            for (int64_t t = H0.rp[i]; t < H0.rp[i + 1]; ++t) dense[(size_t)(i * n0 + H0.ci[t])] = H0.v[t];
        TmpDev<double> buf_a;
        CK(cudaMalloc(&buf_a.p, sizeof(double) * std::max<int64_t>(1, n0 * n0)));
        double *a = buf_a.p;
        CK(h2d(ctx, a, dense.data(), sizeof(double) * n0 * n0));
        const int64_t nbp = (n0 + 31) / 32 * 32;
        if ((st = dalloc(ctx, &ctx->cperm, n0))) return st;
        if ((st = dalloc(ctx, &ctx->ctile, k8_tile_doubles((int)n0)))) return st;
        if ((st = dalloc(ctx, &ctx->crec, k8_rec_doubles((int)n0)))) return st;
        if ((st = dalloc(ctx, &ctx->czf, nbp))) return st;
        if ((st = dalloc(ctx, &ctx->chacc, 2 * nbp))) return st;
        if ((st = dalloc(ctx, &ctx->cb, nbp))) return st;
        if ((st = dalloc(ctx, &ctx->csync, k8_sync_words((int)n0)))) return st;
        CK(cudaMemsetAsync(ctx->csync, 0, sizeof(unsigned long long) * k8_sync_words((int)n0), ctx->stream));
        CK(cudaMemsetAsync(ctx->d_status, 0, sizeof(int), ctx->stream));
        EvTimer tk7(ctx->stream);
        launch_dense_lu(a, (int)n0, ctx->cperm, ctx->d_status, ctx->d_scal, ctx->stream);
        ctx->t_k7 = tk7.stop();
        if ((st = check_launch(ctx))) return st;
        int bad = 0;
        CK(d2h(ctx, &bad, ctx->d_status, sizeof(int)));
        if (bad) return fail(ctx, MHDP_ESINGULAR, "singular coarse operator", -1);
        EvTimer tk8(ctx->stream);
        launch_k8_pack(a, (int)n0, ctx->ctile, ctx->crec, ctx->stream);
        ctx->t_k8pack = tk8.stop();
        if ((st = check_launch(ctx))) return st;
        CK(cudaStreamSynchronize(ctx->stream));
    }
    tick(ctx->t_stage[5]);
    ctx->setup_done = true;
    ctx->t_setup_wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - wall0).count();
    return MHDP_OK;
}

mhdp_status mhdp_setup_timings(const mhdp_ctx *ctx, double *out, int len) {
    if (!ctx || !out || len < 3 + ctx->nlev) return MHDP_EINVAL;
    if (!ctx->setup_done) return MHDP_ESTATE;
    out[0] = ctx->t_k7;
    out[1] = ctx->t_k8pack;
    out[2] = ctx->t_setup_wall;
    for (int l = 0; l < ctx->nlev; ++l) out[3 + l] = ctx->t_k6[l];
    for (int k = 0; k < 6 && 3 + ctx->nlev + k < len; ++k) out[3 + ctx->nlev + k] = ctx->t_stage[k];
    return MHDP_OK;
}

int mhdp_num_levels(const mhdp_ctx *ctx) { return ctx ? ctx->nlev : 0; }

mhdp_status mhdp_get_level_info(const mhdp_ctx *ctx, int level, mhdp_level_info *out) {
    if (!ctx || !out || !valid_level(ctx, level) || !ctx->loaded[level]) return MHDP_EINVAL;
    const HostLevel &H = ctx->H[level];
    memset(out, 0, sizeof(*out));
    out->n = H.n;
    out->nnz = H.rp.empty() ? 0 : H.rp[H.n];
    if (level > 0) {
        const int64_t np = (int64_t)H.pptr.size() - 1;
        out->npatch = np;
        out->sum_n = H.pptr[np];
        for (int64_t i = 0; i < np; ++i) {
            const int64_t k = H.pptr[i + 1] - H.pptr[i];
            out->sum_n2 += k * k;
            out->max_n = std::max<long long>(out->max_n, (long long)k);
        }
        out->p_nnz = H.prp[H.n];
    }
    if (ctx->setup_done) {
        const DevLevel &L = ctx->D[level];
        out->bytes_operator = L.bytes_op;
        out->bytes_factors = level > 0 ? L.bytes_fac : 8LL * k8_tile_doubles(ctx->n0);
        out->bytes_transfer = L.bytes_tr;
    }
    return MHDP_OK;
}

mhdp_status mhdp_spmv(mhdp_ctx *ctx, int level, const double *x_dev, double *y_dev) {
    mhdp_status st = need_setup(ctx);
    if (st) return st;
    if (!valid_level(ctx, level) || !x_dev || !y_dev) return fail(ctx, MHDP_EINVAL, "bad arguments");
    residual(ctx, level, nullptr, x_dev, y_dev);
    return check_launch(ctx);
}

mhdp_status mhdp_residual(mhdp_ctx *ctx, int level, const double *b_dev, const double *x_dev, double *r_dev) {
    mhdp_status st = need_setup(ctx);
    if (st) return st;
    if (!valid_level(ctx, level) || !b_dev || !x_dev || !r_dev) return fail(ctx, MHDP_EINVAL, "bad arguments");
    residual(ctx, level, b_dev, x_dev, r_dev);
    return check_launch(ctx);
}

mhdp_status mhdp_patch_apply(mhdp_ctx *ctx, int level, const double *r_dev) {
    mhdp_status st = need_setup(ctx);
    if (st) return st;
    if (!valid_level(ctx, level) || level < 1 || !r_dev) return fail(ctx, MHDP_EINVAL, "bad arguments");
    launch_patch_apply(ctx->D[level].P, r_dev, ctx->stream);
    return check_launch(ctx);
}

mhdp_status mhdp_patch_update(mhdp_ctx *ctx, int level, double *x_dev) {
    mhdp_status st = need_setup(ctx);
    if (st) return st;
    if (!valid_level(ctx, level) || level < 1 || !x_dev) return fail(ctx, MHDP_EINVAL, "bad arguments");
    launch_patch_update(ctx->D[level].P, ctx->D[level].n, x_dev, 0, ctx->stream);
    return check_launch(ctx);
}

mhdp_status mhdp_smooth(mhdp_ctx *ctx, int level, int nsweeps, int x_is_zero, const double *b_dev, double *x_dev) {
    mhdp_status st = need_setup(ctx);
    if (st) return st;
    if (!valid_level(ctx, level) || level < 1 || nsweeps < 0 || !b_dev || !x_dev)
        return fail(ctx, MHDP_EINVAL, "bad arguments");
    for (int s = 0; s < nsweeps; ++s) sweep(ctx, level, b_dev, x_dev, x_is_zero && s == 0);
    return check_launch(ctx);
}

mhdp_status mhdp_restrict(mhdp_ctx *ctx, int level, const double *r_dev, double *rc_dev) {
    mhdp_status st = need_setup(ctx);
    if (st) return st;
    if (!valid_level(ctx, level) || level < 1 || !r_dev || !rc_dev) return fail(ctx, MHDP_EINVAL, "bad arguments");
    launch_restrict(ctx->D[level].PrT, r_dev, rc_dev, ctx->stream);
    return check_launch(ctx);
}

mhdp_status mhdp_prolong_add(mhdp_ctx *ctx, int level, const double *ec_dev, double *x_dev) {
    mhdp_status st = need_setup(ctx);
    if (st) return st;
    if (!valid_level(ctx, level) || level < 1 || !ec_dev || !x_dev) return fail(ctx, MHDP_EINVAL, "bad arguments");
    launch_prolong_add(ctx->D[level].Pr, ec_dev, x_dev, ctx->stream);
    return check_launch(ctx);
}

// diagnostics: one coarse solve with K8's per-block globaltimer stamps (ns) copied to
// trace_host[(pass * nb + block) * 5 + k], k = claim start, claim+diag staged, chain start,
// chain done (CTA 0), far-warp publish; nb = ceil(n0 / 32).  Synchronises.
mhdp_status mhdp_coarse_solve_trace(mhdp_ctx *ctx, const double *b_dev, double *x_dev, long long *trace_host) {
    mhdp_status st = need_setup(ctx);
    if (st) return st;
    if (!b_dev || !x_dev || !trace_host || b_dev == x_dev) return fail(ctx, MHDP_EINVAL, "bad arguments");
    const int64_t cnt = 32 * (int64_t)((ctx->n0 + 31) / 32);
    TmpDev<long long> tr;
    CK(cudaMalloc(&tr.p, sizeof(long long) * std::max<int64_t>(1, cnt)));
    CK(cudaMemsetAsync(tr.p, 0, sizeof(long long) * std::max<int64_t>(1, cnt), ctx->stream));
    CK(launch_k8_solve(ctx->ctile, ctx->crec, ctx->cperm, ctx->n0, b_dev, x_dev, ctx->czf, ctx->chacc, ctx->csync,
                       ctx->stream, tr.p));
    CK(d2h(ctx, trace_host, tr.p, sizeof(long long) * cnt));
    return check_launch(ctx);
}

mhdp_status mhdp_coarse_solve(mhdp_ctx *ctx, const double *b_dev, double *x_dev) {
    mhdp_status st = need_setup(ctx);
    if (st) return st;
    if (!b_dev || !x_dev) return fail(ctx, MHDP_EINVAL, "bad arguments");
    coarse_solve(ctx, b_dev, x_dev);
    return check_launch(ctx);
}

mhdp_status mhdp_vcycle(mhdp_ctx *ctx, int level, const double *b_dev, double *x_dev) {
    mhdp_status st = need_setup(ctx);
    if (st) return st;
    if (!valid_level(ctx, level) || !b_dev || !x_dev) return fail(ctx, MHDP_EINVAL, "bad arguments");
    if (ctx->graphs_off || ctx->graphs_disabled) {
        vcycle(ctx, level, b_dev, x_dev);
        return check_launch(ctx);
    }
    mhdp_ctx::VGraph *g = nullptr;
    for (auto &e : ctx->graphs)
        if (e.level == level && e.b == b_dev && e.x == x_dev && e.smoother == ctx->p.smoother &&
            e.its == ctx->p.smoother_its)
            g = &e;
    if (!g) {
        mhdp_ctx::VGraph e;
        e.level = level; e.b = b_dev; e.x = x_dev; e.smoother = ctx->p.smoother; e.its = ctx->p.smoother_its;
        if (ctx->graphs.size() >= 16) drop_graphs(ctx);
        ctx->graphs.push_back(e);
        g = &ctx->graphs.back();
    }
    if (g->exec) {
        CK(cudaGraphLaunch(g->exec, ctx->stream));
        g_launches += g->nkern;
        return check_launch(ctx);
    }
    if (g->calls++ == 0) {           // first call: run directly (also initialises kernel attributes)
        vcycle(ctx, level, b_dev, x_dev);
        return check_launch(ctx);
    }
    if ((st = check_launch(ctx))) return st;
    if (!ctx->cap) CK(cudaStreamCreateWithFlags(&ctx->cap, cudaStreamNonBlocking));
    cudaStream_t saved = ctx->stream;
    const long long before = g_launches;
    cudaGraph_t graph = nullptr;
    bool ok = cudaStreamBeginCapture(ctx->cap, cudaStreamCaptureModeThreadLocal) == cudaSuccess;
    if (ok) {
        ctx->stream = ctx->cap;
        vcycle(ctx, level, b_dev, x_dev);
        ctx->stream = saved;
        ok = cudaStreamEndCapture(ctx->cap, &graph) == cudaSuccess && graph;
    }
    cudaGraphExec_t exec = nullptr;
    if (ok) ok = cudaGraphInstantiate(&exec, graph, 0) == cudaSuccess;
    if (graph) cudaGraphDestroy(graph);
    const long long nk = g_launches - before;
    g_launches = before;
    if (!ok) {                       // capture unsupported here: run uncaptured from now on
        cudaGetLastError();
        ctx->graphs_off = true;
        vcycle(ctx, level, b_dev, x_dev);
        return check_launch(ctx);
    }
    g->exec = exec;
    g->nkern = nk;
    CK(cudaGraphLaunch(exec, ctx->stream));
    g_launches += nk;
    return check_launch(ctx);
}

mhdp_status mhdp_vcycle_host(mhdp_ctx *ctx, const double *b_host, double *x_host) {
    mhdp_status st = need_setup(ctx);
    if (st) return st;
    if (!b_host || !x_host) return fail(ctx, MHDP_EINVAL, "bad arguments");
    const int l = ctx->nlev - 1;
    DevLevel &L = ctx->D[l];
    double *db = L.b, *dx = nullptr;
    if (l == 0) dx = L.x;
    else {
        if (!ctx->vh) { if ((st = dalloc(ctx, &ctx->vh, L.n))) return st; }
        dx = ctx->vh;
    }
    CK(cudaMemcpyAsync(db, b_host, sizeof(double) * L.n, cudaMemcpyHostToDevice, ctx->stream));
    vcycle(ctx, l, db, dx);
    CK(cudaMemcpyAsync(x_host, dx, sizeof(double) * L.n, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    return check_launch(ctx);
}

mhdp_status mhdp_vcycle_host_batch(mhdp_ctx *ctx, int nrhs, const double *b_host, double *x_host) {
    mhdp_status st = need_setup(ctx);
    if (st) return st;
    if (nrhs < 0 || (nrhs > 0 && (!b_host || !x_host))) return fail(ctx, MHDP_EINVAL, "bad arguments");
    if (nrhs == 0) return MHDP_OK;
    const int l = ctx->nlev - 1;
    const int64_t n = ctx->D[l].n;
    const size_t bytes = sizeof(double) * (size_t)n;
    for (int t = 0; t < 2; ++t) {
        if (!ctx->hb[t] && (st = dalloc(ctx, &ctx->hb[t], n))) return st;
        if (!ctx->hx[t] && (st = dalloc(ctx, &ctx->hx[t], n))) return st;
    }
    if (!ctx->s_in) {
        CK(cudaStreamCreateWithFlags(&ctx->s_in, cudaStreamNonBlocking));
        CK(cudaStreamCreateWithFlags(&ctx->s_out, cudaStreamNonBlocking));
        CK(cudaEventCreateWithFlags(&ctx->ev_start, cudaEventDisableTiming));
        for (int t = 0; t < 2; ++t) {
            CK(cudaEventCreateWithFlags(&ctx->ev_in[t], cudaEventDisableTiming));
            CK(cudaEventCreateWithFlags(&ctx->ev_done[t], cudaEventDisableTiming));
            CK(cudaEventCreateWithFlags(&ctx->ev_out[t], cudaEventDisableTiming));
        }
    }
    // the copy streams start after the work already queued on the context stream
    CK(cudaEventRecord(ctx->ev_start, ctx->stream));
    CK(cudaStreamWaitEvent(ctx->s_in, ctx->ev_start, 0));
    CK(cudaStreamWaitEvent(ctx->s_out, ctx->ev_start, 0));
    for (int k = 0; k < nrhs; ++k) {
        const int t = k & 1;
        // slot t was last used by right-hand side k - 2: its V-cycle must have read hb[t]
        // before the upload, its download must have read hx[t] before the next V-cycle
        if (k >= 2) CK(cudaStreamWaitEvent(ctx->s_in, ctx->ev_done[t], 0));
        CK(cudaMemcpyAsync(ctx->hb[t], b_host + (int64_t)k * n, bytes, cudaMemcpyHostToDevice, ctx->s_in));
        CK(cudaEventRecord(ctx->ev_in[t], ctx->s_in));
        CK(cudaStreamWaitEvent(ctx->stream, ctx->ev_in[t], 0));
        if (k >= 2) CK(cudaStreamWaitEvent(ctx->stream, ctx->ev_out[t], 0));
        if ((st = mhdp_vcycle(ctx, l, ctx->hb[t], ctx->hx[t]))) {
            // copies of earlier right-hand sides still point into the caller's buffers
            cudaStreamSynchronize(ctx->s_in);
            cudaStreamSynchronize(ctx->s_out);
            return st;
        }
        CK(cudaEventRecord(ctx->ev_done[t], ctx->stream));
        CK(cudaStreamWaitEvent(ctx->s_out, ctx->ev_done[t], 0));
        CK(cudaMemcpyAsync(x_host + (int64_t)k * n, ctx->hx[t], bytes, cudaMemcpyDeviceToHost, ctx->s_out));
        CK(cudaEventRecord(ctx->ev_out[t], ctx->s_out));
    }
    CK(cudaStreamSynchronize(ctx->s_out));
    CK(cudaStreamSynchronize(ctx->stream));
    return check_launch(ctx);
}

mhdp_status mhdp_smooth_host(mhdp_ctx *ctx, int level, int nsweeps, int x_is_zero, const double *b_host,
                             double *x_host) {
    mhdp_status st = need_setup(ctx);
    if (st) return st;
    if (!valid_level(ctx, level) || level < 1 || !b_host || !x_host) return fail(ctx, MHDP_EINVAL, "bad arguments");
    DevLevel &L = ctx->D[level];
    CK(cudaMemcpyAsync(L.b, b_host, sizeof(double) * L.n, cudaMemcpyHostToDevice, ctx->stream));
    if (!x_is_zero) CK(cudaMemcpyAsync(L.x, x_host, sizeof(double) * L.n, cudaMemcpyHostToDevice, ctx->stream));
    for (int s = 0; s < nsweeps; ++s) sweep(ctx, level, L.b, L.x, x_is_zero && s == 0);
    CK(cudaMemcpyAsync(x_host, L.x, sizeof(double) * L.n, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    return check_launch(ctx);
}

mhdp_status mhdp_set_smoother(mhdp_ctx *ctx, int smoother, int smoother_its) {
    if (!ctx) return MHDP_EINVAL;
    if (smoother != 0 && smoother != 1) return fail(ctx, MHDP_EINVAL, "smoother must be 0 or 1");
    if (smoother == 1 && (smoother_its < 1 || smoother_its > 32))
        return fail(ctx, MHDP_EINVAL, "smoother_its must be in 1..32");
    if (smoother == 1 && ctx->setup_done) {
        cudaSetDevice(ctx->device);
        for (int l = 1; l < ctx->nlev; ++l) {
            mhdp_status st = alloc_smoother(ctx, ctx->D[l], smoother_its);
            if (st) return st;
        }
    }
    ctx->p.smoother = smoother;
    ctx->p.smoother_its = smoother_its;
    return MHDP_OK;
}

mhdp_status mhdp_set_graphs(mhdp_ctx *ctx, int enable) {
    if (!ctx) return MHDP_EINVAL;
    ctx->graphs_disabled = !enable;
    return MHDP_OK;
}

int mhdp_vcycle_graphs_active(const mhdp_ctx *ctx) {
    if (!ctx || ctx->graphs_off) return 0;
    int n = 0;
    for (const auto &g : ctx->graphs) n += g.exec != nullptr;
    return n;
}

// Right-preconditioned (F)GMRES on the finest level (c.9): x0 = 0, modified
// Gram-Schmidt (w <- fma(-h, v, w)), v_{k+1} = w / |w|, Givens rotations on the device
// with every product and sum rounded separately, inner products in the R-dot order --
// the oracle's orc_fgmres step for step.  With the Richardson smoother the V-cycle is
// linear and this is GMRES(V) (a8); with the GMRES(6) smoother it is FGMRES (NEXT-1).
// hist (host, optional, maxit + 1): hist[k] = |g_k|, k = 0..its.
mhdp_status krylov_solve(mhdp_ctx *ctx, const double *b_dev, double *x_dev, double rtol, double atol, int maxit,
                         int *its_out, double *relres_out, double *hist) {
    mhdp_status st = need_setup(ctx);
    if (st) return st;
    if (!b_dev || !x_dev || maxit < 1 || maxit > 2000) return fail(ctx, MHDP_EINVAL, "bad arguments");
    const int l = ctx->nlev - 1;
    const int64_t n = ctx->D[l].n;
    cudaStream_t s = ctx->stream;
    if (ctx->f_cap < maxit) {
        if ((st = dalloc(ctx, &ctx->fV, n * (int64_t)(maxit + 1)))) return st;
        if ((st = dalloc(ctx, &ctx->fZ, n * (int64_t)maxit))) return st;
        if ((st = dalloc(ctx, &ctx->fw, n))) return st;
        if ((st = dalloc(ctx, &ctx->fpart, 2 * ((n + 255) / 256) + 2))) return st;
        if ((st = dalloc(ctx, &ctx->fscal, KrylovScal::size(maxit)))) return st;
        ctx->f_cap = maxit;
    }
    const int m = maxit;
    KrylovScal S(ctx->fscal, m);
    CK(cudaMemsetAsync(ctx->fscal, 0, sizeof(double) * KrylovScal::size(m), s));
    double *V = ctx->fV, *Z = ctx->fZ, *w = ctx->fw;
    auto read = [&](const double *p) {
        double v = 0;
        cudaMemcpyAsync(&v, p, sizeof(double), cudaMemcpyDeviceToHost, s);
        cudaStreamSynchronize(s);
        return v;
    };
    launch_dot_pinned(b_dev, b_dev, n, ctx->fpart, S.g, 1, s);
    launch_fill(x_dev, 0.0, n, s);
    const double beta = read(S.g);
    const double tol = std::max(rtol * beta, atol);
    if (hist) hist[0] = beta;
    if (its_out) *its_out = 0;
    if (relres_out) *relres_out = beta > 0 ? 1.0 : 0.0;
    if (beta <= tol) return check_launch(ctx);
    launch_div_dev(V, b_dev, S.g, n, s);
    int k = 0;
    bool conv = false;
    double gk = beta;
    for (k = 0; k < m; ++k) {
        vcycle(ctx, l, V + (int64_t)k * n, Z + (int64_t)k * n);
        residual(ctx, l, nullptr, Z + (int64_t)k * n, w);
        for (int i = 0; i <= k; ++i) {
            launch_dot_pinned(w, V + (int64_t)i * n, n, ctx->fpart, S.H + i * m + k, 0, s);
            launch_axpy_negdev(w, S.H + i * m + k, V + (int64_t)i * n, n, s);
        }
        launch_dot_pinned(w, w, n, ctx->fpart, S.hn + k, 1, s);
        launch_givens(S.H, m, S.cs, S.sn, S.g, S.hn + k, k, nullptr, s);
        gk = std::fabs(read(S.g + k + 1));
        if (hist) hist[k + 1] = gk;
        if (gk <= tol) { ++k; conv = true; break; }
        if (read(S.hn + k) == 0.0) { ++k; break; }
        launch_div_dev(V + (int64_t)(k + 1) * n, w, S.hn + k, n, s);
    }
    launch_backsub(S.H, m, S.g, k, nullptr, S.y, s);
    launch_basis_update(x_dev, Z, n, S.y, k, nullptr, n, s);
    CK(cudaStreamSynchronize(s));
    if (its_out) *its_out = k;
    if (relres_out) *relres_out = gk / beta;
    if ((st = check_launch(ctx))) return st;
    return conv ? MHDP_OK : fail(ctx, MHDP_ENOCONV, "GMRES reached maxit");
}

mhdp_status mhdp_gmres(mhdp_ctx *ctx, const double *b_dev, double *x_dev, double rtol, double atol, int maxit,
                       int *its_out, double *relres_out, double *hist_out) {
    return krylov_solve(ctx, b_dev, x_dev, rtol, atol, maxit, its_out, relres_out, hist_out);
}

mhdp_status mhdp_fgmres(mhdp_ctx *ctx, const double *b_dev, double *x_dev, double rtol, double atol, int maxit,
                        int *its_out, double *relres_out, double *hist_out) {
    return krylov_solve(ctx, b_dev, x_dev, rtol, atol, maxit, its_out, relres_out, hist_out);
}

mhdp_status mhdp_dot(mhdp_ctx *ctx, const double *a_dev, const double *b_dev, long long n, double *out_host) {
    if (!ctx) return MHDP_EINVAL;
    if (ctx->host_only) return fail(ctx, MHDP_ECUDA, "host-only context");
    if (!out_host || n < 0 || (n > 0 && (!a_dev || !b_dev))) return fail(ctx, MHDP_EINVAL, "bad arguments");
    cudaSetDevice(ctx->device);
    double *part = nullptr, *out = nullptr;
    CK(cudaMalloc(&part, sizeof(double) * (2 * ((n + 255) / 256) + 2)));
    CK(cudaMalloc(&out, sizeof(double)));
    launch_dot_pinned(a_dev, b_dev, n, part, out, 0, ctx->stream);
    CK(cudaMemcpyAsync(out_host, out, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    cudaFree(part);
    cudaFree(out);
    return check_launch(ctx);
}

mhdp_status mhdp_export_csr(const mhdp_ctx *ctx, int level, long long *rowptr, int *col, double *val) {
    if (!ctx || !valid_level(ctx, level) || !ctx->loaded[level] || !rowptr || !col || !val) return MHDP_EINVAL;
    const HostLevel &H = ctx->H[level];
    memcpy(rowptr, H.rp.data(), sizeof(int64_t) * (H.n + 1));
    memcpy(col, H.ci.data(), sizeof(int) * H.ci.size());
    memcpy(val, H.v.data(), sizeof(double) * H.v.size());
    return MHDP_OK;
}

mhdp_status mhdp_export_patches(const mhdp_ctx *ctx, int level, long long *pptr, int *pdofs) {
    if (!ctx || !valid_level(ctx, level) || level < 1 || !ctx->loaded[level] || !pptr || !pdofs) return MHDP_EINVAL;
    const HostLevel &H = ctx->H[level];
    memcpy(pptr, H.pptr.data(), sizeof(int64_t) * H.pptr.size());
    memcpy(pdofs, H.pdofs.data(), sizeof(int) * H.pdofs.size());
    return MHDP_OK;
}

mhdp_status mhdp_export_patch_vertices(const mhdp_ctx *ctx, int level, int *verts) {
    if (!ctx || !valid_level(ctx, level) || level < 1 || !ctx->loaded[level] || !verts) return MHDP_EINVAL;
    const HostLevel &H = ctx->H[level];
    const int64_t np = (int64_t)H.pptr.size() - 1;
    if ((int64_t)H.pvert.size() != np) return fail(const_cast<mhdp_ctx *>(ctx), MHDP_ESTATE, "patches not from a mesh");
    memcpy(verts, H.pvert.data(), sizeof(int) * np);
    return MHDP_OK;
}

mhdp_status mhdp_export_prolongation(const mhdp_ctx *ctx, int level, long long *prow, int *pcol, double *pval) {
    if (!ctx || !valid_level(ctx, level) || level < 1 || !ctx->loaded[level] || !prow || !pcol || !pval)
        return MHDP_EINVAL;
    const HostLevel &H = ctx->H[level];
    memcpy(prow, H.prp.data(), sizeof(int64_t) * H.prp.size());
    memcpy(pcol, H.pci.data(), sizeof(int) * H.pci.size());
    memcpy(pval, H.pv.data(), sizeof(double) * H.pv.size());
    return MHDP_OK;
}

mhdp_status mhdp_export_patch_lu(mhdp_ctx *ctx, int level, long long patch, double *lu, int *perm) {
    mhdp_status st = need_setup(ctx);
    if (st) return st;
    if (!valid_level(ctx, level) || level < 1 || !lu || !perm) return fail(ctx, MHDP_EINVAL, "bad arguments");
    const HostLevel &H = ctx->H[level];
    const int64_t np = (int64_t)H.pptr.size() - 1;
    if (patch < 0 || patch >= np) return fail(ctx, MHDP_EINVAL, "bad patch index");
    const DevPatches &P = ctx->D[level].P;
    const int n = (int)(H.pptr[patch + 1] - H.pptr[patch]);
    int64_t foff = 0;
    CK(cudaStreamSynchronize(ctx->stream));
    CK(d2h(ctx, &foff, P.foff + patch, sizeof(int64_t)));
    std::vector<double> pk((size_t)n * n + n);
    CK(d2h(ctx, pk.data(), P.fac + foff, sizeof(double) * (n * n + n)));
    // decode the packed streaming layout (kernels.cu pack_fwd / pack_bwd)
    for (int j = 0; j < n; ++j) {
        const int64_t f = (int64_t)j * n - (int64_t)j * (j + 1) / 2;
        const int64_t b = (int64_t)n * (n - 1) - (int64_t)j * (j + 1) / 2 + 2 * (n - 1 - j);
        for (int i = 0; i < n; ++i)
            lu[(size_t)i * n + j] = i > j ? pk[f + i - j - 1] : (i == j ? pk[b] : pk[b + 2 + i]);
    }
    CK(d2h(ctx, perm, P.perm + H.pptr[patch], sizeof(int) * n));
    return MHDP_OK;
}

mhdp_status mhdp_export_slots(mhdp_ctx *ctx, int level, double *y) {
    mhdp_status st = need_setup(ctx);
    if (st) return st;
    if (!valid_level(ctx, level) || level < 1 || !y) return fail(ctx, MHDP_EINVAL, "bad arguments");
    CK(cudaStreamSynchronize(ctx->stream));
    CK(d2h(ctx, y, ctx->D[level].P.y, sizeof(double) * ctx->D[level].P.sum_n));
    return MHDP_OK;
}

mhdp_status mhdp_synchronize(mhdp_ctx *ctx) {
    if (!ctx) return MHDP_EINVAL;
    if (ctx->host_only) return MHDP_OK;
    CK(cudaSetDevice(ctx->device));
    CK(cudaStreamSynchronize(ctx->stream));
    return check_launch(ctx);
}

mhdp_status mhdp_last_error(const mhdp_ctx *ctx, char *buf, int len, long long *where) {
    if (!ctx) return MHDP_EINVAL;
    if (buf && len > 0) {
        strncpy(buf, ctx->err.c_str(), (size_t)len - 1);
        buf[len - 1] = 0;
    }
    if (where) *where = ctx->where;
    return MHDP_OK;
}

long long mhdp_launch_count(const mhdp_ctx *ctx) { return ctx ? g_launches - ctx->launches0 : 0; }

}  // extern "C"

// =====================================================================================
// NEXT-3: the coupled Newton system over [u | p | E | B] (Table 1) and the
// paper's outer solver: FGMRES with the block upper-triangular preconditioner
//   y_EB = S~^-1 r_EB   (two FGMRES iterations on the E-B block, E-B V-cycle)
//   z_u  = r_u - K y_EB,  K = [J | J~ + D~1 + D~2]
//   y_up = M~^-1 z      (two FGMRES iterations on the (u,p) block, preconditioned by
//                        y_p = -(1/Re + gamma) M_p^-1 s_p, y_u = V_u(s_u - B^T y_p))
// Same operation order as the oracle (reading R-outer); inner products R-dot.
// =====================================================================================
struct mhdp_coupled {
    mhdp_ctx *vel = nullptr, *eb = nullptr;
    bool host_only = true;
    int64_t nu = 0, np = 0, nE = 0, nB = 0, n = 0;
    HostLevel Ah, Muph;           // global operator and the (u,p) block (host copies)
    HostCsr Kh, Bth;
    DevSell A, Mup;
    int64_t *K_rp = nullptr, *Bt_rp = nullptr;
    int *K_ci = nullptr, *Bt_ci = nullptr;
    double *K_v = nullptr, *Bt_v = nullptr;
    double cS = 0, Kinv = 0;
    struct KWs {
        int64_t n = 0;
        int m = 0;
        double *V = nullptr, *Z = nullptr, *w = nullptr, *part = nullptr, *scal = nullptr;
        int *kk = nullptr;
    } Web, Wup, Wout;
    double *z = nullptr, *t = nullptr;
    std::string err;
};

namespace {

mhdp_status kws_alloc(mhdp_ctx *ctx, mhdp_coupled::KWs &W, int64_t n, int m) {
    if (W.m >= m && W.n == n) return MHDP_OK;
    mhdp_status st;
    W.n = n; W.m = m;
    if ((st = dalloc(ctx, &W.V, n * (int64_t)(m + 1)))) return st;
    if ((st = dalloc(ctx, &W.Z, n * (int64_t)m))) return st;
    if ((st = dalloc(ctx, &W.w, n))) return st;
    if ((st = dalloc(ctx, &W.part, 2 * ((n + 255) / 256) + 2))) return st;
    if ((st = dalloc(ctx, &W.scal, KrylovScal::size(m)))) return st;
    if ((st = dalloc(ctx, &W.kk, 1))) return st;
    return MHDP_OK;
}

typedef std::function<void(const double *, double *)> DevOp;

// flexible GMRES on the device (R-outer / fgmres_gen of the oracle).  fixed: exactly m
// iterations, asynchronous, breakdown through the device Krylov dimension; else stop at
// |g_k+1| <= max(rtol |b|, atol) with one scalar read per iteration.
int fgmres_dev(mhdp_ctx *ctx, mhdp_coupled::KWs &W, const DevOp &A, const DevOp &P, const double *b, double *x,
               bool fixed, double rtol, double atol, int m, double *relres, bool *conv_out) {
    cudaStream_t s = ctx->stream;
    const int64_t n = W.n;
    KrylovScal S(W.scal, W.m);
    const int ld = W.m;
    auto read = [&](const double *p) {
        double v = 0;
        cudaMemcpyAsync(&v, p, sizeof(double), cudaMemcpyDeviceToHost, s);
        cudaStreamSynchronize(s);
        return v;
    };
    launch_dot_pinned(b, b, n, W.part, S.g, 1, s);
    launch_fill(x, 0.0, n, s);
    if (fixed) {
        launch_krylov_init(S.g, m, W.kk, s);
        launch_div_dev(W.V, b, S.g, n, s);
        for (int k = 0; k < m; ++k) {
            P(W.V + (int64_t)k * n, W.Z + (int64_t)k * n);
            A(W.Z + (int64_t)k * n, W.w);
            for (int i = 0; i <= k; ++i) {
                launch_dot_pinned(W.w, W.V + (int64_t)i * n, n, W.part, S.H + i * ld + k, 0, s);
                launch_axpy_negdev(W.w, S.H + i * ld + k, W.V + (int64_t)i * n, n, s);
            }
            launch_dot_pinned(W.w, W.w, n, W.part, S.hn + k, 1, s);
            launch_givens(S.H, ld, S.cs, S.sn, S.g, S.hn + k, k, W.kk, s);
            if (k + 1 < m) launch_div_dev(W.V + (int64_t)(k + 1) * n, W.w, S.hn + k, n, s);
        }
        launch_backsub(S.H, ld, S.g, m, W.kk, S.y, s);
        launch_basis_update(x, W.Z, n, S.y, m, W.kk, n, s);
        if (conv_out) *conv_out = true;
        return m;
    }
    const double beta = read(S.g);
    const double tol = std::max(rtol * beta, atol);
    if (relres) *relres = beta > 0 ? 1.0 : 0.0;
    if (conv_out) *conv_out = true;
    if (beta == 0.0 || beta <= tol) return 0;
    launch_div_dev(W.V, b, S.g, n, s);
    int k = 0;
    bool conv = false;
    double gk = beta;
    for (k = 0; k < m; ++k) {
        P(W.V + (int64_t)k * n, W.Z + (int64_t)k * n);
        A(W.Z + (int64_t)k * n, W.w);
        for (int i = 0; i <= k; ++i) {
            launch_dot_pinned(W.w, W.V + (int64_t)i * n, n, W.part, S.H + i * ld + k, 0, s);
            launch_axpy_negdev(W.w, S.H + i * ld + k, W.V + (int64_t)i * n, n, s);
        }
        launch_dot_pinned(W.w, W.w, n, W.part, S.hn + k, 1, s);
        launch_givens(S.H, ld, S.cs, S.sn, S.g, S.hn + k, k, nullptr, s);
        gk = std::fabs(read(S.g + k + 1));
        if (gk <= tol) { ++k; conv = true; break; }
        if (read(S.hn + k) == 0.0) { ++k; break; }
        if (k + 1 < m) launch_div_dev(W.V + (int64_t)(k + 1) * n, W.w, S.hn + k, n, s);
    }
    launch_backsub(S.H, ld, S.g, k, nullptr, S.y, s);
    launch_basis_update(x, W.Z, n, S.y, k, nullptr, n, s);
    if (relres) *relres = gk / beta;
    if (conv_out) *conv_out = conv;
    return k;
}

void coupled_precondition(mhdp_coupled *c, const double *r, double *y) {
    mhdp_ctx *ve = c->vel, *eb = c->eb;
    cudaStream_t s = ve->stream;
    const int te = eb->nlev - 1, tv = ve->nlev - 1;
    const int64_t nup = c->nu + c->np;
    const double *rEB = r + nup;
    double *yEB = y + nup;
    DevOp A_eb = [&](const double *x, double *out) { residual(eb, te, nullptr, x, out); };
    DevOp P_eb = [&](const double *in, double *out) { vcycle(eb, te, in, out); };
    fgmres_dev(ve, c->Web, A_eb, P_eb, rEB, yEB, true, 0, 0, 2, nullptr, nullptr);
    launch_csr_sub(c->nu, c->K_rp, c->K_ci, c->K_v, yEB, r, c->z, s);                 // z_u = r_u - K y_EB
    cudaMemcpyAsync(c->z + c->nu, r + c->nu, sizeof(double) * c->np, cudaMemcpyDeviceToDevice, s);
    DevOp A_up = [&](const double *x, double *out) { launch_residual(c->Mup, nullptr, x, out, s); };
    DevOp P_up = [&](const double *in, double *out) {
        launch_scale2(out + c->nu, in + c->nu, c->cS, c->Kinv, c->np, s);            // y_p
        launch_csr_sub(c->nu, c->Bt_rp, c->Bt_ci, c->Bt_v, out + c->nu, in, c->t, s);   // s_u - B^T y_p
        vcycle(ve, tv, c->t, out);                                                     // y_u
    };
    fgmres_dev(ve, c->Wup, A_up, P_up, c->z, y, true, 0, 0, 2, nullptr, nullptr);
}

void csr_transpose(const HostCsr &A, HostCsr &T) {
    T.n = A.ncols; T.ncols = A.n;
    T.rp.assign(T.n + 1, 0);
    for (int64_t t = 0; t < A.rp[A.n]; ++t) T.rp[A.ci[t] + 1]++;
    for (int64_t j = 0; j < T.n; ++j) T.rp[j + 1] += T.rp[j];
    T.ci.resize(A.rp[A.n]); T.v.resize(A.rp[A.n]);
    std::vector<int64_t> pos(T.rp.begin(), T.rp.end() - 1);
    for (int64_t i = 0; i < A.n; ++i)
        for (int64_t t = A.rp[i]; t < A.rp[i + 1]; ++t) {
            const int64_t q = pos[A.ci[t]]++;
            T.ci[q] = (int)i; T.v[q] = A.v[t];
        }
}

struct RowCat {   // concatenates rows of several CSRs (column shifts) into one CSR
    HostLevel &H;
    explicit RowCat(HostLevel &h, int64_t n) : H(h) { H.n = n; H.rp.assign(1, 0); H.ci.clear(); H.v.clear(); }
    template <class R>
    void push(const R &rp, const std::vector<int> &ci, const std::vector<double> &v, int64_t row, int64_t shift) {
        for (int64_t t = rp[row]; t < rp[row + 1]; ++t) { H.ci.push_back((int)(ci[t] + shift)); H.v.push_back(v[t]); }
    }
    void end() { H.rp.push_back((int64_t)H.ci.size()); }
};

}  // namespace

extern "C" {

void mhdp_coupled_destroy(mhdp_coupled *c) {
    if (!c) return;
    mhdp_destroy(c->vel);
    mhdp_destroy(c->eb);
    delete c;
}

mhdp_status mhdp_coupled_create(mhdp_coupled **out, int cuda_device, void *cuda_stream, const mhdp_mesh *mesh,
                                const mhdp_params *params, const double *w_vertex_host,
                                const double *bn_vertex_host) {
    if (!out || !mesh || !params || !w_vertex_host) return MHDP_EINVAL;
    if (params->degree > 1) return MHDP_EINVAL;   // the k = 2 coupling blocks are not built
    *out = nullptr;
    mhdp_coupled *c = new (std::nothrow) mhdp_coupled();
    if (!c) return MHDP_ENOMEM;
    mhdp_status st;
    if ((st = mhdp_create(&c->vel, cuda_device, cuda_stream)) || (st = mhdp_create(&c->eb, cuda_device, cuda_stream))) {
        mhdp_coupled_destroy(c);
        return st;
    }
    c->host_only = cuda_device < 0;
    if ((st = mhdp_assemble_lorentz(c->vel, MHDP_BLOCK_ALVEL, mesh, params, w_vertex_host, bn_vertex_host)) ||
        (st = mhdp_assemble(c->eb, MHDP_BLOCK_EB, mesh, params, w_vertex_host))) {
        c->err = c->vel->err.empty() ? c->eb->err : c->vel->err;
        *out = c;
        return st;
    }
    CouplingBlocks cb;
    auto rowmax = [](const HostLevel &H, int64_t rows) {
        std::vector<double> m((size_t)rows, 0.0);
        for (int64_t r = 0; r < rows; ++r)
            for (int64_t t = H.rp[r]; t < H.rp[r + 1]; ++t) m[r] = std::max(m[r], std::fabs(H.v[t]));
        return m;
    };
    const HostLevel &Hv = c->vel->H[c->vel->nlev - 1], &He = c->eb->H[c->eb->nlev - 1];
    const std::vector<double> fu = rowmax(Hv, Hv.n), fE = rowmax(He, He.n);   // R-cgrid floors
    std::string e = assemble_coupling(mesh->dim, mesh->n_fine, c->vel->p, w_vertex_host, bn_vertex_host, fu.data(),
                                      fE.data(), cb);
    if (!e.empty()) { c->err = e; *out = c; return MHDP_EINVAL; }
    c->nu = cb.nu; c->np = cb.np; c->nE = cb.nE; c->nB = cb.nB;
    c->n = c->nu + c->np + c->nE + c->nB;
    c->cS = -(1.0 / c->vel->p.Re + c->vel->p.gamma);
    const int N = mesh->n_fine;
    c->Kinv = mesh->dim == 2 ? 2.0 * N * N : 6.0 * (double)N * N * N;
    const HostLevel &Av = c->vel->H[c->vel->nlev - 1], &Ae = c->eb->H[c->eb->nlev - 1];
    HostCsr B;
    csr_transpose(cb.Bt, B);
    const int64_t su = 0, sp = c->nu, sE = c->nu + c->np, sB = sE + c->nE;
    RowCat ga(c->Ah, c->n), gm(c->Muph, c->nu + c->np);
    c->Kh.n = c->nu; c->Kh.ncols = c->nE + c->nB; c->Kh.rp.assign(1, 0);
    for (int64_t i = 0; i < c->nu; ++i) {
        ga.push(Av.rp, Av.ci, Av.v, i, su); ga.push(cb.Bt.rp, cb.Bt.ci, cb.Bt.v, i, sp);
        ga.push(cb.J.rp, cb.J.ci, cb.J.v, i, sE); ga.push(cb.Dt.rp, cb.Dt.ci, cb.Dt.v, i, sB); ga.end();
        gm.push(Av.rp, Av.ci, Av.v, i, 0); gm.push(cb.Bt.rp, cb.Bt.ci, cb.Bt.v, i, c->nu); gm.end();
        for (int64_t t = cb.J.rp[i]; t < cb.J.rp[i + 1]; ++t) { c->Kh.ci.push_back(cb.J.ci[t]); c->Kh.v.push_back(cb.J.v[t]); }
        for (int64_t t = cb.Dt.rp[i]; t < cb.Dt.rp[i + 1]; ++t) {
            c->Kh.ci.push_back((int)(cb.Dt.ci[t] + c->nE)); c->Kh.v.push_back(cb.Dt.v[t]);
        }
        c->Kh.rp.push_back((int64_t)c->Kh.ci.size());
    }
    for (int64_t q = 0; q < c->np; ++q) {
        ga.push(B.rp, B.ci, B.v, q, su); ga.end();
        gm.push(B.rp, B.ci, B.v, q, 0); gm.end();
    }
    for (int64_t r = 0; r < c->nE; ++r) {
        ga.push(cb.G.rp, cb.G.ci, cb.G.v, r, su); ga.push(Ae.rp, Ae.ci, Ae.v, r, sE); ga.end();
    }
    for (int64_t r = 0; r < c->nB; ++r) { ga.push(Ae.rp, Ae.ci, Ae.v, c->nE + r, sE); ga.end(); }
    c->Bth = std::move(cb.Bt);
    *out = c;
    if (c->host_only) return MHDP_OK;
    // device: both hierarchies, the global operator, (u,p) block, K and B^T
    if ((st = mhdp_setup(c->vel)) || (st = mhdp_setup(c->eb))) {
        c->err = c->vel->err.empty() ? c->eb->err : c->vel->err;
        return st;
    }
    mhdp_ctx *ctx = c->vel;
    if ((st = make_sell(ctx, c->Ah, c->A, nullptr))) return st;
    if ((st = make_sell(ctx, c->Muph, c->Mup, nullptr))) return st;
    if ((st = upload(ctx, &c->K_rp, c->Kh.rp.data(), c->nu + 1))) return st;
    if ((st = upload(ctx, &c->K_ci, c->Kh.ci.data(), (int64_t)c->Kh.ci.size()))) return st;
    if ((st = upload(ctx, &c->K_v, c->Kh.v.data(), (int64_t)c->Kh.v.size()))) return st;
    if ((st = upload(ctx, &c->Bt_rp, c->Bth.rp.data(), c->nu + 1))) return st;
    if ((st = upload(ctx, &c->Bt_ci, c->Bth.ci.data(), (int64_t)c->Bth.ci.size()))) return st;
    if ((st = upload(ctx, &c->Bt_v, c->Bth.v.data(), (int64_t)c->Bth.v.size()))) return st;
    if ((st = kws_alloc(ctx, c->Web, c->nE + c->nB, 2))) return st;
    if ((st = kws_alloc(ctx, c->Wup, c->nu + c->np, 2))) return st;
    if ((st = dalloc(ctx, &c->z, c->nu + c->np))) return st;
    if ((st = dalloc(ctx, &c->t, c->nu))) return st;
    CK(cudaStreamSynchronize(ctx->stream));
    return MHDP_OK;
}

mhdp_status mhdp_coupled_sizes(const mhdp_coupled *c, long long *out) {
    if (!c || !out) return MHDP_EINVAL;
    out[0] = c->nu; out[1] = c->np; out[2] = c->nE; out[3] = c->nB; out[4] = c->Ah.rp.empty() ? 0 : c->Ah.rp.back();
    return MHDP_OK;
}

mhdp_status mhdp_coupled_export_csr(const mhdp_coupled *c, long long *rowptr, int *col, double *val) {
    if (!c || !rowptr || !col || !val || c->Ah.rp.empty()) return MHDP_EINVAL;
    memcpy(rowptr, c->Ah.rp.data(), sizeof(int64_t) * c->Ah.rp.size());
    memcpy(col, c->Ah.ci.data(), sizeof(int) * c->Ah.ci.size());
    memcpy(val, c->Ah.v.data(), sizeof(double) * c->Ah.v.size());
    return MHDP_OK;
}

static mhdp_status coupled_ready(mhdp_coupled *c) {
    if (!c) return MHDP_EINVAL;
    if (c->host_only) { c->err = "host-only coupled system"; return MHDP_ECUDA; }
    if (!c->vel->setup_done || !c->eb->setup_done || !c->A.sptr) { c->err = "coupled system not set up"; return MHDP_ESTATE; }
    cudaSetDevice(c->vel->device);
    return MHDP_OK;
}

mhdp_status mhdp_coupled_apply(mhdp_coupled *c, const double *x_dev, double *y_dev) {
    mhdp_status st = coupled_ready(c);
    if (st) return st;
    if (!x_dev || !y_dev) return MHDP_EINVAL;
    launch_residual(c->A, nullptr, x_dev, y_dev, c->vel->stream);
    return check_launch(c->vel);
}

mhdp_status mhdp_coupled_precondition(mhdp_coupled *c, const double *r_dev, double *y_dev) {
    mhdp_status st = coupled_ready(c);
    if (st) return st;
    if (!r_dev || !y_dev) return MHDP_EINVAL;
    coupled_precondition(c, r_dev, y_dev);
    return check_launch(c->vel);
}

mhdp_status mhdp_coupled_fgmres(mhdp_coupled *c, const double *b_dev, double *x_dev, double rtol, double atol,
                                int maxit, int *its_out, double *relres_out) {
    mhdp_status st = coupled_ready(c);
    if (st) return st;
    if (!b_dev || !x_dev || maxit < 1 || maxit > 500) return MHDP_EINVAL;
    mhdp_ctx *ctx = c->vel;
    if ((st = kws_alloc(ctx, c->Wout, c->n, maxit))) { c->err = ctx->err; return st; }
    cudaStream_t s = ctx->stream;
    DevOp A = [&](const double *x, double *y) { launch_residual(c->A, nullptr, x, y, s); };
    DevOp P = [&](const double *r, double *y) { coupled_precondition(c, r, y); };
    double rel = 0;
    bool conv = false;
    const int its = fgmres_dev(ctx, c->Wout, A, P, b_dev, x_dev, false, rtol, atol, maxit, &rel, &conv);
    CK(cudaStreamSynchronize(s));
    if (its_out) *its_out = its;
    if (relres_out) *relres_out = rel;
    if ((st = check_launch(ctx))) return st;
    if (!conv) { c->err = "FGMRES reached maxit"; return MHDP_ENOCONV; }
    return MHDP_OK;
}

mhdp_status mhdp_coupled_set_smoother(mhdp_coupled *c, int smoother, int its) {
    if (!c) return MHDP_EINVAL;
    mhdp_status st = mhdp_set_smoother(c->vel, smoother, its);
    if (!st) st = mhdp_set_smoother(c->eb, smoother, its);
    return st;
}

mhdp_status mhdp_coupled_last_error(const mhdp_coupled *c, char *buf, int len) {
    if (!c || !buf || len <= 0) return MHDP_EINVAL;
    std::string e = !c->err.empty() ? c->err : (!c->vel->err.empty() ? c->vel->err : c->eb->err);
    strncpy(buf, e.c_str(), (size_t)len - 1);
    buf[len - 1] = 0;
    return MHDP_OK;
}

}  // extern "C"
