// brdf_device.cu -- the sm_100a BRDF pipeline behind vrte_compute_brdf.
//
// Stage map (reference -> here):
//   prepare_homogeneous  pipeline.cpp:57-93   -> H: GSF tables, E/F, F*E,
//                                                Hessenberg, Francis QR,
//                                                eigenvectors, mode recovery,
//                                                8N residuals
//   solve_incident/particular pipeline.cpp:122-142 -> P: all incidents x
//                                                4 Stokes channels at once on
//                                                the shared Schur form
//   solve_incident/boundary   pipeline.cpp:145-175 -> B: one real LU per order,
//                                                every (incident, channel) a RHS
//   nodal_components/value    pipeline.cpp:201-220 + brdf.cpp:100-117 -> S
// Everything for one shape lives in a plan whose buffers are reused.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <thread>
#include <type_traits>
#include <vector>

#include "boundary.cuh"
#include "kernels.cuh"
#include "particular.cuh"
#include "refine.cuh"
#include "synth.cuh"
#include "vrte/vrte_cuda.h"

namespace vrte {

[[noreturn]] void cuda_fail(cudaError_t e, const char* what, const char* file, int line) {
    char buf[512];
    std::snprintf(buf, sizeof buf, "CUDA error %s (%s) at %s:%d: %s", cudaGetErrorName(e),
                  cudaGetErrorString(e), file, line, what);
    throw std::runtime_error(buf);
}

namespace {

constexpr double kRefineTarget = 5e-11;  // per-mode 8N residual after refinement
constexpr double kPartTarget = 1e-7;     // particular 8N balance residual (gate 1e-6)
constexpr int kPartExtraMax = 3;

template <typename T>
struct DevBuf {
    T* p = nullptr;
    size_t n = 0;
    void alloc(size_t count) {
        if (count == n && p) return;
        release();
        n = count;
        if (count) VRTE_CUDA_CHECK(cudaMalloc(&p, sizeof(T) * count));
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
    }
    ~DevBuf() { release(); }
    void upload(const T* h, size_t count, cudaStream_t st) {
        alloc(count);
        if (count) VRTE_CUDA_CHECK(cudaMemcpyAsync(p, h, sizeof(T) * count, cudaMemcpyHostToDevice, st));
    }
};

GemmBatch gemm(int m, int n, int k, const double* a, long long lda, long long sa, bool ta,
               const double* b, long long ldb, long long sb, bool tb, double* c, long long ldc,
               long long sc, int batch, double alpha = 1.0, double beta = 0.0) {
    GemmBatch g{};
    g.m = m;
    g.n = n;
    g.k = k;
    g.a = a;
    g.lda = lda;
    g.stride_a = sa;
    g.trans_a = ta;
    g.b = b;
    g.ldb = ldb;
    g.stride_b = sb;
    g.trans_b = tb;
    g.c = c;
    g.ldc = ldc;
    g.stride_c = sc;
    g.batch = batch;
    g.alpha = alpha;
    g.beta = beta;
    return g;
}

}  // namespace
}  // namespace vrte

using namespace vrte;

struct vrte_cuda_plan {
    int device = 0;
    cudaStream_t st = nullptr;
    int Lc = 0;
    int N = 0, L = 0, P = 0, S = 0, n_in = 0, n_dphi = 0, NO = 0, m_begin = 0, m_stride = 1;
    int d = 0, R = 0, G = 0, B = 0;
    int Be = 0;  // slots [0, Be) run the eigen pipeline, [Be, B) are free-streaming (analytic)
    bool full_orders = true;
    bool full_solution = false;  // radiance path: back substitution through every layer
    struct RadBufs {             // radiance.cu scratch, persistent across calls
        DevBuf<double> taus, mus, phis, dtop, dbeam, gsf_o, wp, wm, bb, acc_a, acc_b, bsrc, bout, bbeam, down, bval,
            comp, field, refl;
    } rad;
    ProblemDev pd{};
    // inputs
    DevBuf<double> nodes, weights, mdiag, omega, greek, tau, mu_in, table, beam_rows, post, trig, refl_top, pre;
    int out_lo = 0;
    bool lean = false;  // problem->concurrent: lower-register kernel builds
    bool concurrent = false;  // other plans share the device: no look-ahead streams
    DevBuf<int> medium, order_index, slot_of_order;
    // homogeneous
    DevBuf<double> gsf_n, gsf_b, E, F, T, Z, psi_p, psi_m, tmp1, tmp2, tmp3, tmp4;
    DevBuf<double> X, AL, BE, FB, W2, UT, EU, hwork, Vinv;
    DevBuf<int> ipivV, permV;
    DevBuf<double> wr, wi, femax, nu, nu0, lam, residual, rho, sigma_m, rshift;
    DevBuf<int> flags, kind_m, sidx;
    // particular
    DevBuf<double> sp, sm, fsp, rhs, W, g, eg, feg, zp, zm, mu_eff, sigma;
    DevBuf<int> kind;
    // boundary
    DevBuf<double> lhs, top0, rhs_b, rhs_x, up;
    DevBuf<int> ipiv, perm;
    // boundary residual gate (boundary.cpp:233-257)
    DevBuf<double> lhs0, anorm, bnorm, condm, dX, Xp, Rp, colsum;
    DevBuf<int> colsum_ticket, order_fail, col_refine;
    DevBuf<double> resm, kdump;
    double *dump_kernel = nullptr, *dump_nu = nullptr, *dump_residual = nullptr, *dump_boundary = nullptr;
    int medium0 = 0;
    DevBuf<double> up_save;
    int ldl = 0;  // row stride of [A | B] (+ the probes' b_k in lhs0): G + R + 16
    const double* lhs0_zeroed = nullptr;
    size_t lhs0_zeroed_key = 0;
    int* refine_host = nullptr;  // page-locked copy of DeviceStatus::bnd_refine
    // synthesis
    DevBuf<double> out;
    // device-sharded solves: the gathered stacks of every order (root shard only)
    DevBuf<double> up_all;
    DevBuf<int> slot_all;
    DeviceStatus* status = nullptr;  // pinned host-mapped would be nicer; device + copy
    DevBuf<DeviceStatus> status_buf;
    cudaEvent_t ev[16] = {};
    cudaStream_t st2 = nullptr;          // side stream: independent work overlapped with the main chain
    cudaEvent_t fork[6] = {}, join[6] = {};
    LuLookahead lula;  // the boundary factorization's look-ahead streams (lu.cu)
    DevBuf<double> Qh;          // Hessenberg Q, formed on the side stream under the QR
    cudaEvent_t evq[3] = {};    // reduction done / Q formed / boundary system cleared
    DevBuf<int> lu_snap;
    // the right-hand sides' elimination, deferred off the factorization (lu.cu
    // LuRhsDefer): per-block row-map snapshots / events, its stream and its end
    LuRhsDefer lurd;
    DevBuf<int> lu_rsnap;
    cudaEvent_t rev[32] = {};
    cudaStream_t st3 = nullptr;
    cudaEvent_t evr = nullptr;
    int refine_iters = 1;
    int refine_extra = 2;
    int* count_host = nullptr;  // page-locked: [0] eigen slots still refining, [1] particular slots
    uint64_t part_extra_iters = 0;
    DevBuf<int> slot_on, part_on, counts, slot_list, slot_n, part_list, part_n;
    DevBuf<double> part_slot, part_prev;
    char* stage = nullptr;  // page-locked staging for the per-call inputs (one async copy each)
    size_t stage_bytes = 0;
    uint64_t launches = 0;
    ~vrte_cuda_plan() {
        if (count_host) cudaFreeHost(count_host);
        if (refine_host) cudaFreeHost(refine_host);
        if (stage) cudaFreeHost(stage);
        for (auto& e : ev)
            if (e) cudaEventDestroy(e);
        for (auto* es : {fork, join})
            for (int i = 0; i < 6; ++i)
                if (es[i]) cudaEventDestroy(es[i]);
        for (auto& e : lula.ev)
            if (e) cudaEventDestroy(e);
        for (auto& e : evq)
            if (e) cudaEventDestroy(e);
        for (auto& e : rev)
            if (e) cudaEventDestroy(e);
        if (evr) cudaEventDestroy(evr);
        if (st3) cudaStreamDestroy(st3);
        if (lula.hi) cudaStreamDestroy(lula.hi);
        if (lula.lo) cudaStreamDestroy(lula.lo);
        if (st2) cudaStreamDestroy(st2);
        if (st) cudaStreamDestroy(st);
    }
};

namespace {


void fill_message(vrte_cuda_result* r, int status, const std::string& msg) {
    if (!r) return;
    r->status = status;
    std::snprintf(r->message, sizeof r->message, "%s", msg.c_str());
}

void check_problem(const vrte_cuda_problem* p) {
    if (!p || p->N < 1 || p->L < 1 || p->n_layers < 1 || p->n_media < 1 || p->n_in < 1 ||
        p->n_dphi < 1)
        throw std::invalid_argument("vrte_cuda: invalid problem dimensions");
    if (4 * p->N > 1024) throw std::invalid_argument("vrte_cuda: N > 256 not supported");
    if (p->base_type == 2 && p->table_n < p->N)
        throw std::invalid_argument("vrte_cuda: mueller table smaller than the quadrature");
}

void setup_plan(vrte_cuda_plan& pl, const vrte_cuda_problem* p) {
    check_problem(p);
    pl.device = p->device;
    if (pl.device >= 0) VRTE_CUDA_CHECK(cudaSetDevice(pl.device));
    if (!pl.st) {
        // the main chain at the highest priority: side-stream work (Q formation,
        // beam source, particular stage) fills the SMs it leaves free
        int lo_prio = 0, hi_prio = 0;
        VRTE_CUDA_CHECK(cudaDeviceGetStreamPriorityRange(&lo_prio, &hi_prio));
        VRTE_CUDA_CHECK(cudaStreamCreateWithPriority(&pl.st, cudaStreamNonBlocking, hi_prio));
    }
    for (auto& e : pl.evq)
        if (!e) VRTE_CUDA_CHECK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    for (auto& e : pl.rev)
        if (!e) VRTE_CUDA_CHECK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    if (!pl.evr) VRTE_CUDA_CHECK(cudaEventCreateWithFlags(&pl.evr, cudaEventDisableTiming));
    if (!pl.st3) VRTE_CUDA_CHECK(cudaStreamCreateWithFlags(&pl.st3, cudaStreamNonBlocking));
    for (auto& e : pl.ev)
        if (!e) VRTE_CUDA_CHECK(cudaEventCreate(&e));
    if (!pl.st2) VRTE_CUDA_CHECK(cudaStreamCreateWithFlags(&pl.st2, cudaStreamNonBlocking));
    for (auto* es : {pl.fork, pl.join})
        for (int i = 0; i < 6; ++i)
            if (!es[i]) VRTE_CUDA_CHECK(cudaEventCreateWithFlags(&es[i], cudaEventDisableTiming));
    if (!pl.lula.hi) {
        int lo_prio = 0, hi_prio = 0;
        VRTE_CUDA_CHECK(cudaDeviceGetStreamPriorityRange(&lo_prio, &hi_prio));
        VRTE_CUDA_CHECK(cudaStreamCreateWithPriority(&pl.lula.hi, cudaStreamNonBlocking, hi_prio));
        VRTE_CUDA_CHECK(cudaStreamCreateWithPriority(&pl.lula.lo, cudaStreamNonBlocking, lo_prio));
        for (auto& e : pl.lula.ev) VRTE_CUDA_CHECK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    if (!pl.count_host) VRTE_CUDA_CHECK(cudaMallocHost(&pl.count_host, 2 * sizeof(int)));
    if (!pl.refine_host) VRTE_CUDA_CHECK(cudaMallocHost(&pl.refine_host, sizeof(int)));
    pl.counts.alloc(2);
    pl.N = p->N;
    pl.L = p->L;
    pl.Lc = p->L_coeffs > 0 ? p->L_coeffs : p->L;
    pl.P = p->n_layers;
    pl.S = p->n_media;
    pl.n_in = p->n_in;
    pl.n_dphi = p->n_dphi;
    pl.full_orders = p->n_orders <= 0;
    pl.NO = pl.full_orders ? p->L : p->n_orders;
    pl.m_begin = pl.full_orders ? 0 : p->m_begin;
    pl.m_stride = pl.full_orders ? 1 : p->m_stride;
    pl.d = 4 * pl.N;
    pl.R = 4 * pl.n_in;
    pl.G = 2 * pl.d * pl.P;
    pl.B = pl.S * pl.NO;
    {
        // trailing free-streaming orders of the last medium: zero kernel for
        // m >= its last nonzero expansion coefficient (or omega = 0)
        const int s = pl.S - 1;
        int lc = 0;
        if (p->omega[s] != 0.0)
            for (int l = 0; l < pl.Lc; ++l)
                for (int q = 0; q < 6; ++q)
                    if (p->greek[((size_t)s * pl.Lc + l) * 6 + q] != 0.0) lc = l + 1;
        int tail = 0;
        for (int mo = pl.NO - 1; mo >= 0; --mo) {
            if (pl.m_begin + mo * pl.m_stride < lc) break;
            ++tail;
        }
        pl.Be = std::max(1, pl.B - tail);  // at least one slot through the pipeline (no empty launches)
        // the lean QR build only pays when the clusters oversubscribe the SMs: concurrent
        // plans of this size, or one plan with more matrices than SM pairs (C4': 256);
        // small order shards and C3 (67 matrices, 134 SMs) keep the faster 225-register build
        int dev = 0, sms = 148;
        if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        pl.lean = (p->concurrent != 0 && 2 * pl.Be >= sms / 2) || 2 * pl.Be > sms;  // (or alone but > 1 wave)
        pl.concurrent = p->concurrent != 0;
    }
    const int N = pl.N, L = pl.L, d = pl.d, R = pl.R, G = pl.G, B = pl.B, NO = pl.NO;
    cudaStream_t st = pl.st;

    std::vector<double> mdiag(d);
    for (int i = 0; i < d; ++i) mdiag[i] = p->nodes[i / 4];
    std::vector<int> medium(p->medium, p->medium + pl.P);
    std::vector<int> order_index(B), slot(L, -1);
    for (int s = 0; s < pl.S; ++s)
        for (int mo = 0; mo < NO; ++mo) order_index[s * NO + mo] = pl.m_begin + mo * pl.m_stride;
    for (int mo = 0; mo < NO; ++mo) {
        const int m = pl.m_begin + mo * pl.m_stride;
        if (m < L) slot[m] = mo;
    }
    // inputs through a page-locked staging area: every H2D copy is truly asynchronous
    // (pageable sources would be staged by the driver one copy at a time)
    {
        const size_t tab_n = p->base_type == 2 ? (size_t)p->table_n * p->table_n * 16 : 16;
        const size_t need_d = 2 * (size_t)N + d + pl.S + (size_t)pl.S * pl.Lc * 6 + pl.P + pl.n_in + tab_n + 32 * (size_t)N +
                              (size_t)pl.n_in * N * 16 + (size_t)pl.n_in * 16 + (size_t)L * pl.n_dphi * 2;
        const size_t need = need_d * sizeof(double) + ((size_t)pl.P + B + L) * sizeof(int) + 32 * 256;
        if (pl.stage_bytes < need) {
            if (pl.stage) cudaFreeHost(pl.stage);
            VRTE_CUDA_CHECK(cudaMallocHost(reinterpret_cast<void**>(&pl.stage), need));
            pl.stage_bytes = need;
        }
    }
    size_t off = 0;
    auto put = [&](auto& buf, const auto* h, size_t n) {
        using T = std::remove_pointer_t<decltype(buf.p)>;
        buf.alloc(n);
        if (!n) return;
        std::memcpy(pl.stage + off, h, sizeof(T) * n);
        VRTE_CUDA_CHECK(cudaMemcpyAsync(buf.p, pl.stage + off, sizeof(T) * n, cudaMemcpyHostToDevice, st));
        off += (sizeof(T) * n + 255) & ~size_t(255);
    };
    put(pl.nodes, p->nodes, N);
    put(pl.weights, p->weights, N);
    put(pl.mdiag, mdiag.data(), d);
    put(pl.omega, p->omega, pl.S);
    put(pl.greek, p->greek, (size_t)pl.S * pl.Lc * 6);
    put(pl.tau, p->tau, pl.P);
    put(pl.medium, medium.data(), pl.P);
    put(pl.mu_in, p->mu_in, pl.n_in);
    if (p->base_type == 2)
        put(pl.table, p->table, (size_t)p->table_n * p->table_n * 16);
    else
        pl.table.alloc(16);
    put(pl.beam_rows, p->beam_rows, (size_t)pl.n_in * N * 16);
    put(pl.post, p->post, (size_t)pl.n_in * 16);
    put(pl.trig, p->trig, (size_t)L * pl.n_dphi * 2);
    pl.out_lo = p->refl_top ? p->out_lo : 0;
    pl.dump_kernel = p->dump_kernel;
    pl.dump_nu = p->dump_nu;
    pl.dump_residual = p->dump_residual;
    pl.dump_boundary = p->dump_boundary;
    pl.medium0 = p->medium[0];
    if (p->refl_top) {
        put(pl.refl_top, p->refl_top, (size_t)N * 16);
        put(pl.pre, p->pre, (size_t)N * 16);
    }
    put(pl.order_index, order_index.data(), B);
    put(pl.slot_of_order, slot.data(), L);

    const size_t dd = (size_t)d * d;
    pl.gsf_n.alloc((size_t)L * pl.Lc * 3 * N);
    pl.gsf_b.alloc((size_t)L * pl.Lc * 3 * pl.n_in);
    for (auto* b : {&pl.E, &pl.F, &pl.T, &pl.Z, &pl.psi_p, &pl.psi_m, &pl.tmp1, &pl.tmp2, &pl.tmp3,
                    &pl.tmp4, &pl.X})
        b->alloc(B * dd);
    for (auto* b : {&pl.AL, &pl.BE, &pl.FB, &pl.W2, &pl.UT, &pl.EU}) b->alloc(2 * B * dd);
    pl.hwork.alloc((size_t)B * hessenberg_work_doubles(d));
    pl.Qh.alloc((size_t)B * d * d);
    pl.Vinv.alloc(B * dd);
    pl.ipivV.alloc((size_t)B * d);
    pl.permV.alloc((size_t)B * d);
    pl.rho.alloc((size_t)B * d * 2);
    pl.sigma_m.alloc((size_t)B * d * 4);
    pl.kind_m.alloc((size_t)B * d * 2);
    pl.sidx.alloc((size_t)B * d);
    pl.rshift.alloc((size_t)B * d);
    pl.wr.alloc((size_t)B * d);
    pl.wi.alloc((size_t)B * d);
    pl.femax.alloc(B);
    pl.nu.alloc((size_t)B * d * 2);
    pl.nu0.alloc((size_t)B * d * 2);
    pl.lam.alloc((size_t)B * d * 2);
    pl.residual.alloc((size_t)B * d);
    pl.flags.alloc((size_t)B * d);
    for (auto* b : {&pl.slot_on, &pl.part_on, &pl.slot_list, &pl.part_list}) b->alloc(B);
    pl.slot_n.alloc(1);
    pl.part_n.alloc(1);
    pl.part_slot.alloc(B);
    pl.part_prev.alloc(B);
    const size_t bdr = (size_t)B * d * R;
    for (auto* b : {&pl.sp, &pl.sm, &pl.fsp, &pl.rhs, &pl.W, &pl.g, &pl.eg, &pl.feg, &pl.zp, &pl.zm})
        b->alloc(bdr);
    pl.mu_eff.alloc((size_t)B * pl.n_in);
    pl.sigma.alloc((size_t)B * R * 2);
    pl.kind.alloc((size_t)B * R);
    pl.ldl = G + R + 16;  // >= G + R + kBndProbes, rows stay 128-byte aligned
    pl.lhs.alloc((size_t)NO * G * pl.ldl);   // augmented [A | B | probes] per order, row-major
    pl.lhs0.alloc((size_t)NO * G * pl.ldl);  // its untouched copy (residual gate)
    pl.Xp.alloc((size_t)NO * G * kBndProbes);
    pl.Rp.alloc((size_t)NO * G * kBndProbes);
    const size_t zkey = ((size_t)G << 40) ^ ((size_t)pl.ldl << 20) ^ (size_t)NO ^ ((size_t)pl.P << 60);
    if (pl.lhs0_zeroed != pl.lhs0.p || pl.lhs0_zeroed_key != zkey) {  // its zero blocks are never written
        VRTE_CUDA_CHECK(cudaMemsetAsync(pl.lhs0.p, 0, sizeof(double) * pl.lhs0.n, st));
        pl.lhs0_zeroed = pl.lhs0.p;
        pl.lhs0_zeroed_key = zkey;
    }
    pl.anorm.alloc((size_t)NO * 2);
    pl.bnorm.alloc((size_t)NO * R * 2);
    pl.condm.alloc((size_t)NO);
    pl.colsum.alloc((size_t)NO * G);
    pl.order_fail.alloc((size_t)NO);
    pl.resm.alloc((size_t)NO);
    pl.col_refine.alloc((size_t)NO * R);
    pl.colsum_ticket.alloc((size_t)NO * ((G + 255) / 256));
    pl.dX.alloc((size_t)NO * G * R);
    pl.top0.alloc((size_t)NO * d * 2 * d);
    pl.rhs_x.alloc((size_t)NO * R * G);
    pl.ipiv.alloc((size_t)NO * G);
    pl.perm.alloc((size_t)NO * G);
    pl.lu_snap.alloc((size_t)NO * G);
    pl.lula.snap = pl.lu_snap.p;
    if (lu_outer_blocks(G) > 32) throw std::invalid_argument("vrte_cuda: boundary system with more than 32 outer blocks");
    pl.lu_rsnap.alloc((size_t)lu_outer_blocks(G) * NO * G);
    pl.lurd.snaps = pl.lu_rsnap.p;
    pl.lurd.ev = pl.rev;
    pl.lurd.nblocks = lu_outer_blocks(G);
    pl.up.alloc((size_t)NO * R * d);
    pl.out.alloc((size_t)pl.n_in * (N - pl.out_lo) * pl.n_dphi * 16);
    pl.status_buf.alloc(1);
    pl.status = pl.status_buf.p;

    ProblemDev& pd = pl.pd;
    pd.N = N;
    pd.L = L;
    pd.Lc = pl.Lc;
    pd.n_media = pl.S;
    pd.n_layers = pl.P;
    pd.n_in = pl.n_in;
    pd.n_dphi = pl.n_dphi;
    pd.n_orders = NO;
    pd.m_begin = pl.m_begin;
    pd.m_stride = pl.m_stride;
    pd.nodes = pl.nodes.p;
    pd.weights = pl.weights.p;
    pd.omega = pl.omega.p;
    pd.greek = pl.greek.p;
    pd.tau = pl.tau.p;
    pd.medium = pl.medium.p;
    pd.mu_in = pl.mu_in.p;
    pd.base_type = p->base_type;
    pd.rho = p->rho;
    pd.table_n = p->table_n;
    pd.table = pl.table.p;
    pd.beam_rows = pl.beam_rows.p;
    pd.refl_top = p->refl_top ? pl.refl_top.p : nullptr;
}

BndArgs make_bnd(vrte_cuda_plan& pl) {
    BndArgs ba{};
    ba.p = pl.pd;
    ba.d = pl.d;
    ba.psi_p = pl.psi_p.p;
    ba.psi_m = pl.psi_m.p;
    ba.nu = pl.nu.p;
    ba.wi = pl.wi.p;
    ba.zp = pl.zp.p;
    ba.zm = pl.zm.p;
    ba.lhs = pl.lhs.p;
    ba.top0 = pl.top0.p;
    // the right-hand sides ride in the LU as columns G .. G+R, the residual
    // probes after them (BRDF path; the radiance path checks every column)
    ba.K = pl.full_solution ? 0 : kBndProbes;
    ba.ldl = ba.ldr = pl.ldl;
    ba.sl = ba.sr = (long long)pl.G * pl.ldl;
    ba.rhs = pl.lhs.p + pl.G;
    ba.up = pl.up.p;
    ba.lhs0 = pl.lhs0.p;
    ba.anorm = pl.anorm.p;
    ba.bnorm = pl.bnorm.p;
    ba.condm = pl.condm.p;
    ba.colsum = pl.colsum.p;
    ba.colsum_ticket = reinterpret_cast<unsigned*>(pl.colsum_ticket.p);
    ba.order_fail = pl.order_fail.p;
    ba.col_refine = pl.col_refine.p;
    ba.resm = pl.resm.p;
    return ba;
}

// The reference's gate on the full solution rhs_x (boundary.cpp:233-257):
// |A x - b| against 1e-10 scale, one refinement step for the right-hand sides
// above it, then 1e-9 scale.  Host-synchronous (the refinement is rare).
int boundary_full_gate(vrte_cuda_plan& pl, const BndArgs& ba, cudaStream_t st) {
    const int G = pl.G, R = pl.R, NO = pl.NO;
    int nl = 2;
    VRTE_CUDA_CHECK(cudaMemsetAsync(&pl.status->max_boundary_residual, 0, sizeof(double), st));
    VRTE_CUDA_CHECK(cudaMemsetAsync(pl.condm.p, 0, sizeof(double) * NO, st));
    VRTE_CUDA_CHECK(cudaMemsetAsync(pl.resm.p, 0, sizeof(double) * NO, st));
    launch_bnd_residual(ba, pl.rhs_x.p, G, R, false, st);
    launch_bnd_check(ba, pl.rhs_x.p, G, R, 0, pl.status, st);
    VRTE_CUDA_CHECK(cudaMemcpyAsync(pl.refine_host, &pl.status->bnd_refine, sizeof(int), cudaMemcpyDeviceToHost, st));
    VRTE_CUDA_CHECK(cudaStreamSynchronize(st));
    if (*pl.refine_host) {
        launch_bnd_refine_rhs(ba, pl.perm.p, pl.dX.p, G, R, st);
        lu_solve_gathered(pl.lhs.p, G, pl.ldl, NO, pl.perm.p, pl.dX.p, R, st);
        launch_bnd_add(ba, pl.rhs_x.p, pl.dX.p, G, R, st);
        launch_bnd_residual(ba, pl.dX.p, G, R, true, st);
        VRTE_CUDA_CHECK(cudaMemsetAsync(&pl.status->max_boundary_residual, 0, sizeof(double), st));
        VRTE_CUDA_CHECK(cudaMemsetAsync(pl.condm.p, 0, sizeof(double) * NO, st));
        VRTE_CUDA_CHECK(cudaMemsetAsync(pl.resm.p, 0, sizeof(double) * NO, st));
        launch_bnd_check(ba, pl.rhs_x.p, G, R, 1, pl.status, st);
        const int one = 1;
        VRTE_CUDA_CHECK(cudaMemcpyAsync(&pl.status->bnd_refined, &one, sizeof(int), cudaMemcpyHostToDevice, st));
        nl += 6 + 4 * ((G + 63) / 64);
    }
    return nl;
}

// up = Z+ of the top layer + Top0 [A_0; B_0]: layer 0's unknowns are the last
// 2d rows of the row-major solution (bnd_col), read column-major as their transpose.
int boundary_top(vrte_cuda_plan& pl, const BndArgs& ba, cudaStream_t st) {
    const int d = pl.d, R = pl.R, G = pl.G;
    launch_copy_zp0(ba, st);
    gemm_batched(gemm(d, R, 2 * d, pl.top0.p, d, (long long)d * 2 * d, false,
                      pl.rhs_x.p + (size_t)(G - 2 * d) * R, R, (long long)G * R, true, pl.up.p, d, (long long)d * R,
                      pl.NO, 1.0, 1.0),
                 st);
    return 2;
}

int run_synth(vrte_cuda_plan& pl, cudaStream_t st) {
    SynthArgs sa{};
    sa.N = pl.N;
    sa.L = pl.L;
    sa.n_in = pl.n_in;
    sa.n_dphi = pl.n_dphi;
    sa.up = pl.up.p;
    sa.slot_of_order = pl.slot_of_order.p;
    sa.trig = pl.trig.p;
    sa.post = pl.post.p;
    sa.out = pl.out.p;
    sa.status = pl.status;
    sa.pre = pl.pd.refl_top ? pl.pre.p : nullptr;
    sa.out_lo = pl.out_lo;
    launch_synth(sa, st);
    return 1;
}

// The device pipeline; returns the number of kernel launches issued.
uint64_t run_pipeline(vrte_cuda_plan& pl, bool synth) {
    const int N = pl.N, L = pl.L, d = pl.d, R = pl.R, G = pl.G, NO = pl.NO;
    const int B = pl.Be;  // eigen / particular batch (free-streaming slots filled analytically)
    const long long dd = (long long)d * d, dR = (long long)d * R;
    cudaStream_t st = pl.st;
    const ProblemDev& pd = pl.pd;
    uint64_t nl = 0;
    pl.part_extra_iters = 0;
    VRTE_CUDA_CHECK(cudaMemsetAsync(pl.status, 0, sizeof(DeviceStatus), st));
    VRTE_CUDA_CHECK(cudaEventRecord(pl.ev[0], st));
    // ---------------- homogeneous
    launch_gsf(pd, pl.nodes.p, N, 1.0, pl.gsf_n.p, st);
    launch_gsf(pd, pl.mu_in.p, pl.n_in, -1.0, pl.gsf_b.p, st);
    if (pl.dump_kernel) {  // debug dump of layer 0's kernel blocks (kernel.cpp:188-214)
        pl.kdump.alloc((size_t)NO * N * N * 32);
        launch_kernel_dump(pd, pl.gsf_n.p, pl.medium0, pl.kdump.p, st);
        ++nl;
    }
    // the beam source terms (particular.cpp:7-25) need only the GSF tables: side stream,
    // overlapped with the homogeneous stage
    cudaStream_t st2 = pl.st2;
    VRTE_CUDA_CHECK(cudaEventRecord(pl.fork[0], st));
    VRTE_CUDA_CHECK(cudaStreamWaitEvent(st2, pl.fork[0], 0));
    launch_beam_source(pd, pl.gsf_n.p, pl.gsf_b.p, pl.sp.p, pl.sm.p, st2);
    VRTE_CUDA_CHECK(cudaEventRecord(pl.join[0], st2));
    launch_build_ef(pd, pl.gsf_n.p, pl.E.p, pl.F.p, st);
    gemm_batched(gemm(d, d, d, pl.F.p, d, dd, false, pl.E.p, d, dd, false, pl.T.p, d, dd, B), st);
    launch_max_abs(pl.T.p, dd, B, pl.femax.p, st);
    VRTE_CUDA_CHECK(cudaEventRecord(pl.ev[5], st));
    // Hessenberg reduction; its Q (independent of the reduced matrix) is formed on
    // the side stream while the QR runs from Z = I on the main stream, and the
    // eigenvectors are X = Q (Z Y)
    launch_hessenberg_reduce(pl.T.p, pl.hwork.p, d, B, st);
    VRTE_CUDA_CHECK(cudaEventRecord(pl.evq[0], st));
    VRTE_CUDA_CHECK(cudaStreamWaitEvent(st2, pl.evq[0], 0));
    launch_hessenberg_formq(pl.Qh.p, pl.hwork.p, d, B, st2);
    VRTE_CUDA_CHECK(cudaEventRecord(pl.evq[1], st2));
    // also under the QR (latency-bound, it leaves bandwidth and 14 SMs): F s+ of the
    // particular right-hand side (F and the beam source only) and the boundary
    // systems' zero fill (the factorization fills them in)
    gemm_batched(gemm(d, R, d, pl.F.p, d, dd, false, pl.sp.p, d, dR, false, pl.fsp.p, d, dR, B), st2);
    launch_bnd_zero(make_bnd(pl), st2);
    VRTE_CUDA_CHECK(cudaEventRecord(pl.evq[2], st2));
    launch_set_identity(pl.Z.p, d, B, st);
    nl += hessenberg_launch_count(d) + 2;
    VRTE_CUDA_CHECK(cudaEventRecord(pl.ev[6], st));
    launch_hqr(pl.T.p, pl.Z.p, pl.wr.p, pl.wi.p, d, B, pl.status, st, nullptr, pl.lean);
    VRTE_CUDA_CHECK(cudaEventRecord(pl.ev[7], st));
    launch_trevc(pl.T.p, pl.wr.p, pl.wi.p, pl.tmp1.p, d, B, st);
    VRTE_CUDA_CHECK(cudaEventRecord(pl.ev[8], st));
    gemm_batched(gemm(d, d, d, pl.Z.p, d, dd, false, pl.tmp1.p, d, dd, false, pl.tmp3.p, d, dd, B), st);
    VRTE_CUDA_CHECK(cudaStreamWaitEvent(st, pl.evq[1], 0));
    gemm_batched(gemm(d, d, d, pl.Qh.p, d, dd, false, pl.tmp3.p, d, dd, false, pl.X.p, d, dd, B), st);
    launch_normalize_modes(pl.X.p, pl.wi.p, d, B, st);
    {
        // V^-1 of the packed eigenvector matrix: the shifted solves of the
        // refinement and of the particular stage run in the eigenbasis
        // (two GEMMs + an independent 1x1/2x2 solve per entry).
        // The column-major V read row-major is V^T: factor V^T, solve V^T Y = I
        // row-major, and Y read column-major is V^-1.
        // Side stream: overlapped with E X, the mode recovery and the first refinement
        // GEMMs (they touch neither the Hessenberg work (Vlu, identity), Vinv nor the V
        // pivots); joined at the first eigenbasis solve.
        double* Vlu = pl.hwork.p;  // Hessenberg work is free again
        VRTE_CUDA_CHECK(cudaEventRecord(pl.fork[1], st));
        VRTE_CUDA_CHECK(cudaStreamWaitEvent(st2, pl.fork[1], 0));
        VRTE_CUDA_CHECK(cudaMemcpyAsync(Vlu, pl.X.p, sizeof(double) * B * dd, cudaMemcpyDeviceToDevice, st2));
        double* Ident = pl.hwork.p + (size_t)B * dd;  // second half of the Hessenberg work (>= 2 d^2 per slot)
        launch_set_identity(Ident, d, B, st2);
        lu_factor_rm(Vlu, d, B, pl.ipivV.p, pl.permV.p, pl.status, pl.order_index.p, st2);
        lu_solve_rm(Vlu, d, B, pl.permV.p, Ident, pl.Vinv.p, d, st2);
        VRTE_CUDA_CHECK(cudaEventRecord(pl.join[1], st2));
        nl += 1 + lu_rm_launch_count(d);
    }
    gemm_batched(gemm(d, d, d, pl.E.p, d, dd, false, pl.X.p, d, dd, false, pl.tmp3.p, d, dd, B), st);
    ModeArgs ma{};
    ma.d = d;
    ma.batch = B;
    ma.wr = pl.wr.p;
    ma.wi = pl.wi.p;
    ma.femax = pl.femax.p;
    ma.X = pl.X.p;
    ma.EX = pl.tmp3.p;
    ma.mdiag = pl.mdiag.p;
    ma.nu = pl.nu.p;
    ma.lam = pl.lam.p;
    ma.flags = pl.flags.p;
    ma.psi_p = pl.psi_p.p;
    ma.psi_m = pl.psi_m.p;
    ma.ab_sum = pl.tmp1.p;
    ma.ab_dif = pl.tmp4.p;
    ma.status = pl.status;
    ma.order_index = pl.order_index.p;
    launch_modes(ma, st);
    // (F E - sigma_c) y_c = r_c for `ncol` columns in place of W = R (ld d):
    // eigenbasis (default) or Schur form.  `out` = Q y (+ beta out).
    bool vinv_joined = false;
    // the refinement's extra steps run their GEMMs on the compacted list of the
    // slots still above target (slot_list / slot_n, set below); main stream only
    const int* zl = nullptr;
    const int* zn = nullptr;
    const int* zl2 = nullptr;  // the particular stage's extra steps (side stream)
    const int* zn2 = nullptr;
    auto mgemm = [&](GemmBatch g, cudaStream_t ss) {
        g.zmap = ss == st ? zl : zl2;
        g.zcount = ss == st ? zn : zn2;
        gemm_batched(g, ss);
    };
    auto shifted_solve = [&](const double* Rm, double* Wm, int ncol, long long wst, const double* sig,
                             const int* knd, double* out, double beta, cudaStream_t ss) {
        if (ss == st && !vinv_joined) {  // V^-1 comes from the side stream: join at its first use
            VRTE_CUDA_CHECK(cudaStreamWaitEvent(st, pl.join[1], 0));
            vinv_joined = true;
        }
        mgemm(gemm(d, ncol, d, pl.Vinv.p, d, dd, false, Rm, d, wst, false, Wm, d, wst, B), ss);
        launch_eig_diag_solve(Wm, d, ncol, wst, pl.wr.p, pl.wi.p, sig, knd, B, ss);
        mgemm(gemm(d, ncol, d, pl.X.p, d, dd, false, Wm, d, wst, false, out, d, wst, B, 1.0, beta), ss);
    };
    auto residual_gemms = [&]() {
        mgemm(gemm(d, d, d, pl.E.p, d, dd, false, pl.tmp1.p, d, dd, false, pl.tmp3.p, d, dd, B), st);
        mgemm(gemm(d, d, d, pl.F.p, d, dd, false, pl.tmp4.p, d, dd, false, pl.tmp2.p, d, dd, B), st);
    };
    // ---------------- particular (particular.cpp:27-107) on the side stream: it needs
    // V^-1 (queued before it there), the beam source and the modes' nu, none of which
    // the refinement below touches except nu -- snapshotted here.  Joined before the
    // boundary stage.
    VRTE_CUDA_CHECK(cudaMemcpyAsync(pl.nu0.p, pl.nu.p, sizeof(double) * 2 * (size_t)B * d, cudaMemcpyDeviceToDevice,
                                    st));
    VRTE_CUDA_CHECK(cudaEventRecord(pl.fork[2], st));
    VRTE_CUDA_CHECK(cudaStreamWaitEvent(st2, pl.fork[2], 0));
    PartArgs pa{};
    pa.d = d;
    pa.batch = B;
    pa.n_in = pl.n_in;
    pa.mu_in = pl.mu_in.p;
    pa.nu = pl.nu0.p;  // the modes' nu before refinement (the refinement updates nu concurrently)
    pa.femax = pl.femax.p;
    pa.mdiag = pl.mdiag.p;
    pa.order_index = pl.order_index.p;
    pa.mu_eff = pl.mu_eff.p;
    pa.sigma = pl.sigma.p;
    pa.kind = pl.kind.p;
    pa.fsp = pl.fsp.p;
    pa.sp = pl.sp.p;
    pa.sm = pl.sm.p;
    pa.rhs = pl.rhs.p;
    pa.g = pl.g.p;
    pa.eg = pl.eg.p;
    pa.feg = pl.feg.p;
    pa.zp = pl.zp.p;
    pa.zm = pl.zm.p;
    pa.status = pl.status;
    launch_dither(pa, st2);
    launch_part_rhs(pa, st2);
    shifted_solve(pl.rhs.p, pl.W.p, R, dR, pl.sigma.p, pl.kind.p, pl.g.p, 0.0, st2);
    gemm_batched(gemm(d, R, d, pl.E.p, d, dd, false, pl.g.p, d, dR, false, pl.eg.p, d, dR, B), st2);
    gemm_batched(gemm(d, R, d, pl.F.p, d, dd, false, pl.eg.p, d, dR, false, pl.feg.p, d, dR, B), st2);
    // Iterative refinement against the true operator F (E g): the Schur form
    // carries a normwise backward error ~eps|FE| that the reference's dense LU
    // (componentwise-small on this graded matrix) does not.
    // One step normally suffices; the interim balance residual (the 8N check of
    // particular.cpp:86-105) decides about more below, at the refinement's host sync.
    // part_on: every slot refines in the first step; the per-slot decision after
    // each interim residual (launch_part_decide) masks the later ones
    pa.part_on = pl.part_on.p;
    pa.part_slot = pl.part_slot.p;
    pa.part_prev = pl.part_prev.p;
    launch_fill_int(pl.part_on.p, B, 1, st2);
    VRTE_CUDA_CHECK(cudaMemsetAsync(pl.part_slot.p, 0, sizeof(double) * B, st2));
    auto part_iteration = [&](bool first) {
        if (!first) {  // the extra steps: GEMMs only on the slots still refining
            launch_compact_slots(pl.part_on.p, B, pl.part_list.p, pl.part_n.p, st2);
            zl2 = pl.part_list.p;
            zn2 = pl.part_n.p;
            nl += 1;
        }
        launch_part_refine_residual(pa, pl.fsp.p, st2);
        shifted_solve(pl.fsp.p, pl.W.p, R, dR, pl.sigma.p, pl.kind.p, pl.g.p, 1.0, st2);
        mgemm(gemm(d, R, d, pl.E.p, d, dd, false, pl.g.p, d, dR, false, pl.eg.p, d, dR, B), st2);
        mgemm(gemm(d, R, d, pl.F.p, d, dd, false, pl.eg.p, d, dR, false, pl.feg.p, d, dR, B), st2);
        zl2 = zn2 = nullptr;
        launch_zpm(pa, st2);
        launch_part_residual(pa, st2, false);
        launch_part_decide(pa, kPartTarget, first, pl.counts.p + 1, st2);
        VRTE_CUDA_CHECK(cudaMemcpyAsync(pl.count_host + 1, pl.counts.p + 1, sizeof(int), cudaMemcpyDeviceToHost, st2));
        VRTE_CUDA_CHECK(cudaEventRecord(pl.join[5], st2));
        nl += 9;
    };
    part_iteration(true);
    nl += 7;
    // (the 8N residual of the unrefined modes is not needed: every refinement
    // step starts by recomputing it, and final_residual() feeds the gate)
    ResidualArgs ra{};
    ra.d = d;
    ra.batch = B;
    ra.wi = pl.wi.p;
    ra.nu = pl.nu.p;
    ra.psi_p = pl.psi_p.p;
    ra.psi_m = pl.psi_m.p;
    ra.G1 = pl.tmp3.p;
    ra.G2 = pl.tmp2.p;
    ra.mdiag = pl.mdiag.p;
    ra.residual = pl.residual.p;
    nl += 11;
    // ---- eigenpair refinement (replaces the polish of homogeneous.cpp:216-268)
    RefineArgs rf{};
    rf.d = d;
    rf.batch = B;
    rf.wi = pl.wi.p;
    rf.mdiag = pl.mdiag.p;
    rf.flags = pl.flags.p;
    rf.wr = pl.wr.p;
    rf.femax = pl.femax.p;
    rf.shift = pl.rshift.p;
    rf.nu = pl.nu.p;
    rf.rho = pl.rho.p;
    rf.psi_p = pl.psi_p.p;
    rf.psi_m = pl.psi_m.p;
    rf.ab_sum = pl.tmp1.p;
    rf.ab_dif = pl.tmp4.p;
    rf.G1 = pl.tmp3.p;
    rf.G2 = pl.tmp2.p;
    rf.sidx = pl.sidx.p;
    rf.AL = pl.AL.p;
    rf.BE = pl.BE.p;
    rf.FB = pl.FB.p;
    rf.UT = pl.UT.p;
    rf.EU = pl.EU.p;
    rf.sigma = pl.sigma_m.p;
    rf.kind = pl.kind_m.p;
    const long long d2 = 2 * dd;
    VRTE_CUDA_CHECK(cudaEventRecord(pl.ev[9], st));
    launch_nu_rho(rf, true, st);
    launch_refine_shift(rf, st);
    auto refine_iteration = [&]() {
        launch_refine_normalize(rf, st);
        residual_gemms();
        launch_refine_setup(rf, st);
        mgemm(gemm(d, 2 * d, d, pl.F.p, d, dd, false, pl.BE.p, d, d2, false, pl.FB.p, d, d2, B), st);
        launch_refine_rhs(rf, st);
        shifted_solve(pl.FB.p, pl.W2.p, 2 * d, d2, pl.sigma_m.p, pl.kind_m.p, pl.UT.p, 0.0, st);
        mgemm(gemm(d, 2 * d, d, pl.E.p, d, dd, false, pl.UT.p, d, d2, false, pl.EU.p, d, d2, B), st);
        launch_refine_update(rf, st);
        nl += 11;
    };
    auto final_residual = [&]() {
        launch_nu_rho(rf, false, st);
        launch_refine_normalize(rf, st);
        residual_gemms();
        launch_residual(ra, st);
        nl += 6;
    };
    for (int it = 0; it < pl.refine_iters; ++it) refine_iteration();
    final_residual();
    // Adaptive: one Newton step normally brings every mode below 1e-11 (the
    // eigenbasis correction is accurate to ~eps |FE| / gap); slots above
    // kRefineTarget refine again (at most refine_extra times; the others are
    // masked, so a slot's result does not depend on the rest of the plan)
    // before the 1e-9 gate in finish().
    launch_fill_int(pl.slot_on.p, B, 1, st);
    rf.slot_on = pl.slot_on.p;
    for (int extra = 0; extra < pl.refine_extra; ++extra) {
        launch_refine_slots(d, B, pl.residual.p, kRefineTarget, pl.slot_on.p, pl.counts.p, st);
        VRTE_CUDA_CHECK(cudaMemcpyAsync(pl.count_host, pl.counts.p, sizeof(int), cudaMemcpyDeviceToHost, st));
        VRTE_CUDA_CHECK(cudaStreamSynchronize(st));
        nl += 2;
        if (*pl.count_host == 0) break;
        launch_compact_slots(pl.slot_on.p, B, pl.slot_list.p, pl.slot_n.p, st);
        zl = pl.slot_list.p;
        zn = pl.slot_n.p;
        refine_iteration();
        final_residual();
        nl += 1;
    }
    zl = zn = nullptr;
    rf.slot_on = nullptr;
    VRTE_CUDA_CHECK(cudaEventRecord(pl.ev[10], st));
    VRTE_CUDA_CHECK(cudaEventRecord(pl.ev[1], st));
    // ---------------- particular: runs on the side stream, concurrent with the refinement;
    // the free-streaming slots' analytic modes and (zero) particular vectors here
    launch_free_modes(d, pl.Be, pl.B, pl.mdiag.p, pl.psi_p.p, pl.psi_m.p, pl.nu.p, pl.wr.p, pl.wi.p,
                      pl.residual.p, pl.zp.p, pl.zm.p, R, st);
    VRTE_CUDA_CHECK(cudaEventRecord(pl.ev[2], st));
    // ---------------- boundary
    const BndArgs ba = make_bnd(pl);
    VRTE_CUDA_CHECK(cudaMemsetAsync(pl.resm.p, 0, sizeof(double) * NO, st));
    VRTE_CUDA_CHECK(cudaStreamWaitEvent(st, pl.evq[2], 0));
    launch_bnd_assemble(ba, st, true);
    // (the right-hand sides need the modes, the free-streaming slots' particular
    // vectors and the assembled system: all queued on the main stream by now)
    VRTE_CUDA_CHECK(cudaEventRecord(pl.fork[3], st));
    // The system matrix is factored as soon as it is assembled: its right-hand
    // sides wait for the particular stage (side stream) and are eliminated on a
    // third stream block by block behind the factorization (lu.cu LuRhsDefer:
    // the same arithmetic as carrying them along).  Look-ahead only for a plan
    // alone on its device: with plans in flight the other plans fill the SMs
    // the look-ahead would, at twice the launches.
    VRTE_CUDA_CHECK(cudaEventRecord(pl.ev[11], st));
    const int K = ba.K, ldl = ba.ldl;
    lu_factor_rm(pl.lhs.p, G, NO, pl.ipiv.p, pl.perm.p, pl.status, pl.order_index.p, st, d, pl.P, ldl, G, nullptr,
                 pl.concurrent ? nullptr : &pl.lula, &pl.lurd);
    // The particular stage's refinement, like the eigenpairs': another step while
    // its balance residual exceeds kPartTarget (a tenth of the reference's 1e-6
    // gate); decided here, with the factorization already queued.
    // Per slot: stops when a step no longer halves the residual (its fp64 floor).
    for (int part_extra = 0; part_extra < kPartExtraMax; ++part_extra) {
        VRTE_CUDA_CHECK(cudaEventSynchronize(pl.join[5]));
        if (pl.count_host[1] == 0) break;
        ++pl.part_extra_iters;
        part_iteration(false);
    }
    launch_part_residual(pa, st2);  // the reference's gates on the final particular vectors
    VRTE_CUDA_CHECK(cudaEventRecord(pl.join[2], st2));
    nl += 1;
    // right-hand sides on the side stream once the particular vectors are there
    VRTE_CUDA_CHECK(cudaStreamWaitEvent(st2, pl.fork[3], 0));
    launch_bnd_rhs(ba, st2);
    VRTE_CUDA_CHECK(cudaEventRecord(pl.join[3], st2));
    // matrix norms of the untouched copy, under the factorization
    launch_bnd_norms(ba, G, R, st2);
    VRTE_CUDA_CHECK(cudaMemsetAsync(pl.condm.p, 0, sizeof(double) * NO, st2));
    VRTE_CUDA_CHECK(cudaEventRecord(pl.join[0], st2));
    nl += 4;
    // their elimination, each block's as soon as both it and the right-hand sides exist
    VRTE_CUDA_CHECK(cudaStreamWaitEvent(pl.st3, pl.join[3], 0));
    lu_rhs_forward(pl.lhs.p, G, ldl, R, NO, pl.lurd, d, pl.P, pl.st3);
    VRTE_CUDA_CHECK(cudaEventRecord(pl.evr, pl.st3));
    VRTE_CUDA_CHECK(cudaStreamWaitEvent(st, pl.evr, 0));
    nl += lu_rhs_forward_launch_count(G);
    VRTE_CUDA_CHECK(cudaEventRecord(pl.ev[12], st));
    if (pl.full_solution) {
        // radiance: every layer's coefficients, under the reference's exact gate
        lu_backsolve_aug(pl.lhs.p, G, ldl, R, NO, pl.perm.p, pl.rhs_x.p, 0, st);
        VRTE_CUDA_CHECK(cudaEventRecord(pl.ev[13], st));
        VRTE_CUDA_CHECK(cudaStreamWaitEvent(st, pl.join[0], 0));
        nl += lu_aug_launch_count(G, 0, 0) + boundary_full_gate(pl, ba, st);
    } else {
        // BRDF: layer 0's unknowns only (the last 2d rows); the K residual probes
        // through every row on the side stream, concurrently
        VRTE_CUDA_CHECK(cudaMemsetAsync(pl.order_fail.p, 0, sizeof(int) * NO, st));
        launch_bnd_probe_setup(ba, pl.perm.p, pl.Xp.p, G, R, st);
        VRTE_CUDA_CHECK(cudaEventRecord(pl.fork[4], st));
        VRTE_CUDA_CHECK(cudaStreamWaitEvent(st2, pl.fork[4], 0));
        lu_few_solve(pl.lhs.p, G, ldl, NO, pl.perm.p, pl.Xp.p, K, kBndCombProbes, st2);
        VRTE_CUDA_CHECK(cudaEventRecord(pl.join[4], st2));
        const int row_lo = G - 2 * d;
        lu_backsolve_aug(pl.lhs.p, G, ldl, R, NO, pl.perm.p, pl.rhs_x.p, row_lo, st);
        VRTE_CUDA_CHECK(cudaEventRecord(pl.ev[13], st));
        VRTE_CUDA_CHECK(cudaStreamWaitEvent(st, pl.join[0], 0));
        VRTE_CUDA_CHECK(cudaStreamWaitEvent(st, pl.join[4], 0));
        launch_bnd_probe_check(ba, pl.Xp.p, pl.Rp.p, pl.rhs_x.p, (row_lo / 64) * 64, G, R, pl.status, st);
        nl += lu_aug_launch_count(G, 0, row_lo) + 1 + 1 + 3;
    }
    nl += boundary_top(pl, ba, st);
    VRTE_CUDA_CHECK(cudaEventRecord(pl.ev[3], st));
    // ---------------- synthesis
    if (synth) nl += run_synth(pl, st);
    VRTE_CUDA_CHECK(cudaEventRecord(pl.ev[4], st));
    return nl;
}

// A residual probe failed (or a solution entry is not finite): the full
// solution of every right-hand side under the reference's exact gate, then the
// tau = 0 stacks and the synthesis again.  Synchronizes the plan's stream;
// returns true when it ran.
std::atomic<int> g_force_fallback{0};

bool boundary_fallback(vrte_cuda_plan& pl, bool synth) {
    if (pl.full_solution) return false;
    if (g_force_fallback.load()) {  // test hook: every order "failed"
        const int one = 1;
        VRTE_CUDA_CHECK(cudaMemcpyAsync(&pl.status->bnd_fallback, &one, sizeof(int), cudaMemcpyHostToDevice, pl.st));
        launch_fill_int(pl.order_fail.p, pl.NO, 1, pl.st);
    }
    VRTE_CUDA_CHECK(cudaMemcpyAsync(pl.refine_host, &pl.status->bnd_fallback, sizeof(int), cudaMemcpyDeviceToHost, pl.st));
    VRTE_CUDA_CHECK(cudaStreamSynchronize(pl.st));
    if (!*pl.refine_host) return false;
    cudaStream_t st = pl.st;
    const BndArgs ba = make_bnd(pl);
    pl.up_save.alloc(pl.up.n);
    VRTE_CUDA_CHECK(cudaMemcpyAsync(pl.up_save.p, pl.up.p, sizeof(double) * pl.up.n, cudaMemcpyDeviceToDevice, st));
    launch_bnd_gather_b(ba, pl.perm.p, pl.rhs_x.p, pl.G, pl.R, st);
    lu_solve_gathered(pl.lhs.p, pl.G, pl.ldl, pl.NO, pl.perm.p, pl.rhs_x.p, pl.R, st);
    uint64_t nl = 1 + lu_rm_launch_count(pl.G);
    nl += boundary_full_gate(pl, ba, st);
    nl += boundary_top(pl, ba, st);
    launch_bnd_keep_passed(ba, pl.up_save.p, st);  // only the failed orders change
    nl += 1;
    if (synth) {
        VRTE_CUDA_CHECK(cudaMemsetAsync(&pl.status->clamped, 0, sizeof(unsigned long long), st));
        VRTE_CUDA_CHECK(cudaMemsetAsync(&pl.status->neg_key, 0, sizeof(unsigned long long), st));
        nl += run_synth(pl, st);
    }
    pl.launches += nl;
    return true;
}

std::string describe_failure(const DeviceStatus& s, const std::vector<double>& residual, int d,
                             const std::vector<int>& order_index) {
    char buf[400];
    switch (s.code) {
        case kFailHqrNoConverge:
            std::snprintf(buf, sizeof buf, "eigen decomposition failed at order m = %d",
                          order_index.empty() ? s.index : order_index[s.index]);
            break;
        case kFailNonFiniteEigen:
            std::snprintf(buf, sizeof buf, "non-finite eigenvalue at order m = %d", s.index);
            break;
        case kFailNegativeAxis:
            std::snprintf(buf, sizeof buf,
                          "eigenvalue on the negative real axis at order m = %d (lambda = %g)",
                          s.index, s.value);
            break;
        case kFailParticular:
            std::snprintf(buf, sizeof buf, "singular beam-response system at order m = %d, mu0 = %g",
                          s.index, s.value);
            break;
        case kFailLuSingular:
            std::snprintf(buf, sizeof buf,
                          "boundary system ill-conditioned at order m = %d (singular pivot at %g)",
                          s.index, s.value);
            break;
        case kFailBoundary:  // boundary.cpp:251-253
            std::snprintf(buf, sizeof buf, "boundary system ill-conditioned at order m = %d (condition ~ %g, residual %g)",
                          s.index, s.value2, s.value);
            break;
        case kFailBalance:  // particular.cpp:101-104
            std::snprintf(buf, sizeof buf, "beam-response residual %g at order m = %d", s.value, s.index);
            break;
        case kFailNonFiniteTable:
            std::snprintf(buf, sizeof buf, "brdf: non-finite table entry (index %d)", s.index);
            break;
        case kFailNegativeIntensity:
            std::snprintf(buf, sizeof buf, "brdf: negative intensity entry %f", s.value);
            break;
        default:
            std::snprintf(buf, sizeof buf, "device failure code %d", s.code);
    }
    (void)residual;
    (void)d;
    return buf;
}

// Post-run host checks: device failure record and the eigen residual bound
// (homogeneous.cpp:280-285).  Fills the result block.
int finish(vrte_cuda_plan& pl, vrte_cuda_result* r) {
    DeviceStatus s{};
    VRTE_CUDA_CHECK(cudaMemcpyAsync(&s, pl.status, sizeof s, cudaMemcpyDeviceToHost, pl.st));
    std::vector<double> res((size_t)pl.B * pl.d);
    VRTE_CUDA_CHECK(cudaMemcpyAsync(res.data(), pl.residual.p, sizeof(double) * res.size(),
                                    cudaMemcpyDeviceToHost, pl.st));
    VRTE_CUDA_CHECK(cudaStreamSynchronize(pl.st));
    std::vector<int> oi((size_t)pl.B);
    for (int s2 = 0; s2 < pl.S; ++s2)
        for (int mo = 0; mo < pl.NO; ++mo) oi[s2 * pl.NO + mo] = pl.m_begin + mo * pl.m_stride;
    double maxres = 0.0;
    int worst = -1;
    for (int b = 0; b < pl.B; ++b)
        for (int j = 0; j < pl.d; ++j) {
            const double v = res[(size_t)b * pl.d + j];
            if (!(v <= maxres)) {
                maxres = v;
                worst = b;
            }
        }
    if (r) {
        float ms = 0;
        cudaEventElapsedTime(&ms, pl.ev[0], pl.ev[1]);
        r->t_homogeneous = ms * 1e-3;
        cudaEventElapsedTime(&ms, pl.ev[1], pl.ev[2]);
        r->t_particular = ms * 1e-3;
        cudaEventElapsedTime(&ms, pl.ev[2], pl.ev[3]);
        r->t_boundary = ms * 1e-3;
        cudaEventElapsedTime(&ms, pl.ev[3], pl.ev[4]);
        r->t_synthesis = ms * 1e-3;
        auto span = [&](int a, int b) {
            float t = 0;
            cudaEventElapsedTime(&t, pl.ev[a], pl.ev[b]);
            return t * 1e-3;
        };
        r->t_device = span(0, 4);
        r->t_hessenberg = span(5, 6);
        r->t_hqr = span(6, 7);
        r->t_trevc = span(7, 8);
        r->t_refine = span(9, 10);
        r->t_lu_factor = span(11, 12);
        r->t_lu_solve = span(12, 13);
        r->dithered = s.dithered;
        r->clamped = s.clamped;
        r->polished = s.polished;
        r->qr_sweeps = s.qr_sweeps;
        r->qr_steps = s.qr_steps;
        for (int q = 0; q < 8; ++q) r->qr_cycles[q] = s.qr_cycles[q];
        r->max_eigen_residual = maxres;
        r->max_particular_residual = s.max_particular_residual;
        r->max_balance_residual = s.max_balance_residual;
        r->max_boundary_residual = s.max_boundary_residual;
        r->boundary_refined = s.bnd_refined ? 1 : 0;
        r->boundary_fallback = s.bnd_fallback ? 1 : 0;
        r->particular_extra_steps = pl.part_extra_iters;
        std::vector<double> cm((size_t)pl.NO);
        VRTE_CUDA_CHECK(cudaMemcpy(cm.data(), pl.condm.p, sizeof(double) * cm.size(), cudaMemcpyDeviceToHost));
        r->max_boundary_condition = 0.0;
        r->boundary_cond_warnings = 0;
        for (double c : cm) {
            r->max_boundary_condition = std::max(r->max_boundary_condition, c);
            if (c > 1e14) ++r->boundary_cond_warnings;
        }
        r->kernel_launches = pl.launches;
        r->eigen_slots = pl.Be;
        r->slots = pl.B;
    }
    // debug dumps (host buffers of the problem)
    if (pl.dump_kernel && pl.kdump.p)
        VRTE_CUDA_CHECK(cudaMemcpy(pl.dump_kernel, pl.kdump.p, sizeof(double) * pl.kdump.n, cudaMemcpyDeviceToHost));
    if (pl.dump_nu)
        VRTE_CUDA_CHECK(cudaMemcpy(pl.dump_nu, pl.nu.p, sizeof(double) * 2 * (size_t)pl.B * pl.d,
                                   cudaMemcpyDeviceToHost));
    if (pl.dump_residual) std::memcpy(pl.dump_residual, res.data(), sizeof(double) * res.size());
    if (pl.dump_boundary) {
        std::vector<double> cm((size_t)pl.NO), rm((size_t)pl.NO);
        VRTE_CUDA_CHECK(cudaMemcpy(cm.data(), pl.condm.p, sizeof(double) * cm.size(), cudaMemcpyDeviceToHost));
        VRTE_CUDA_CHECK(cudaMemcpy(rm.data(), pl.resm.p, sizeof(double) * rm.size(), cudaMemcpyDeviceToHost));
        for (int mo = 0; mo < pl.NO; ++mo) {
            pl.dump_boundary[2 * mo] = cm[mo];
            pl.dump_boundary[2 * mo + 1] = rm[mo];
        }
    }
    if (s.code == kFailNegativeIntensity && s.neg_key != 0) {
        const unsigned long long idx = ~s.neg_key;  // first offending entry, reference order
        VRTE_CUDA_CHECK(cudaMemcpy(&s.value, pl.out.p + idx * 16, sizeof(double), cudaMemcpyDeviceToHost));
    }
    if (s.code != 0) {
        fill_message(r, 3, describe_failure(s, res, pl.d, oi));
        return 3;
    }
    if (!(maxres <= kEigenResidualBound)) {
        char buf[256];
        std::snprintf(buf, sizeof buf, "homogeneous mode residual %g exceeds %g at order m = %d",
                      maxres, kEigenResidualBound, worst >= 0 ? oi[worst] : -1);
        fill_message(r, 3, buf);
        return 3;
    }
    if (r) {
        r->status = 0;
        r->message[0] = 0;
    }
    return 0;
}

template <typename Fn>
int32_t guarded(vrte_cuda_result* r, Fn&& fn) {
    try {
        return fn();
    } catch (const std::invalid_argument& e) {
        fill_message(r, 5, e.what());
        return 5;
    } catch (const std::exception& e) {
        fill_message(r, 3, e.what());
        return 3;
    }
}

}  // namespace

namespace {
// Plan pool: every concurrent caller leases its own plan (device buffers +
// stream), so the entry points stay reentrant, and plans outlive the calling
// thread -- a batch's short-lived worker threads reuse them instead of
// re-allocating gigabytes per call (a thread_local cache dies with its thread).
std::mutex g_pool_mu;
std::vector<std::unique_ptr<vrte_cuda_plan>> g_pool;
std::vector<int> g_pool_dev;

struct PlanLease {
    std::unique_ptr<vrte_cuda_plan> p;
    int dev = 0;
    explicit PlanLease(int device) {
        dev = device;
        if (dev < 0) VRTE_CUDA_CHECK(cudaGetDevice(&dev));
        std::lock_guard<std::mutex> lk(g_pool_mu);
        for (size_t i = g_pool.size(); i-- > 0;)
            if (g_pool_dev[i] == dev) {
                p = std::move(g_pool[i]);
                g_pool.erase(g_pool.begin() + i);
                g_pool_dev.erase(g_pool_dev.begin() + i);
                return;
            }
        p = std::make_unique<vrte_cuda_plan>();
    }
    ~PlanLease() {
        if (!p) return;
        std::lock_guard<std::mutex> lk(g_pool_mu);
        g_pool.push_back(std::move(p));
        g_pool_dev.push_back(dev);
    }
    vrte_cuda_plan& operator*() { return *p; }
};
}  // namespace

namespace {
std::mutex g_host_mu;
std::vector<std::pair<size_t, void*>> g_host_free;  // (bytes, pinned block)
std::vector<void*> g_heap_blocks;                    // blocks that fell back to the heap
}  // namespace

extern "C" {

void* vrte_cuda_host_alloc(size_t bytes) {
    if (bytes == 0) bytes = 8;
    {
        std::lock_guard<std::mutex> lk(g_host_mu);
        for (size_t i = g_host_free.size(); i-- > 0;)
            if (g_host_free[i].first == bytes) {
                void* p = g_host_free[i].second;
                g_host_free.erase(g_host_free.begin() + i);
                return p;
            }
    }
    void* p = nullptr;
    if (cudaMallocHost(&p, bytes) != cudaSuccess) {
        cudaGetLastError();  // clear; no device: plain heap memory
        p = std::malloc(bytes);
        if (!p) throw std::bad_alloc();
        std::lock_guard<std::mutex> lk(g_host_mu);
        g_heap_blocks.push_back(p);
    }
    return p;
}

void vrte_cuda_host_free(void* p, size_t bytes) {
    if (!p) return;
    if (bytes == 0) bytes = 8;
    std::lock_guard<std::mutex> lk(g_host_mu);
    for (size_t i = 0; i < g_heap_blocks.size(); ++i)
        if (g_heap_blocks[i] == p) {
            g_heap_blocks.erase(g_heap_blocks.begin() + i);
            std::free(p);
            return;
        }
    if (g_host_free.size() >= 64) {  // bound the cache
        cudaFreeHost(g_host_free.front().second);
        g_host_free.erase(g_host_free.begin());
    }
    g_host_free.emplace_back(bytes, p);
}

void vrte_cuda_debug_force_boundary_fallback(int32_t on) { g_force_fallback.store(on != 0); }

int32_t vrte_cuda_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
    return n;
}

int32_t vrte_cuda_current_device(void) {
    int d = 0;
    if (cudaGetDevice(&d) != cudaSuccess) return 0;
    return d;
}

int32_t vrte_cuda_plan_create(const vrte_cuda_problem* problem, vrte_cuda_plan** out,
                              vrte_cuda_result* result) {
    return guarded(result, [&]() -> int32_t {
        if (!out) throw std::invalid_argument("null plan pointer");
        *out = nullptr;
        auto pl = std::make_unique<vrte_cuda_plan>();
        setup_plan(*pl, problem);
        pl->launches = run_pipeline(*pl, pl->full_orders);
        boundary_fallback(*pl, pl->full_orders);
        const int rc = finish(*pl, result);
        if (rc == 0) *out = pl.release();  // a failed plan frees its device buffers here
        return rc;
    });
}

int32_t vrte_cuda_plan_acquire(const vrte_cuda_problem* problem, vrte_cuda_plan** out, vrte_cuda_result* result) {
    return guarded(result, [&]() -> int32_t {
        if (!out || !problem) throw std::invalid_argument("null plan pointer");
        *out = nullptr;
        PlanLease lease(problem->device);
        vrte_cuda_plan& pl = *lease;
        setup_plan(pl, problem);
        pl.full_solution = false;
        pl.launches = run_pipeline(pl, pl.full_orders);
        boundary_fallback(pl, pl.full_orders);
        const int rc = finish(pl, result);
        if (rc == 0) *out = lease.p.release();  // the caller's until vrte_cuda_plan_release
        return rc;
    });
}

void vrte_cuda_plan_release(vrte_cuda_plan* pl) {
    if (!pl) return;
    std::unique_ptr<vrte_cuda_plan> p(pl);
    int dev = pl->device;
    if (dev < 0 && cudaGetDevice(&dev) != cudaSuccess) dev = 0;
    std::lock_guard<std::mutex> lk(g_pool_mu);
    g_pool.push_back(std::move(p));
    g_pool_dev.push_back(dev);
}

int32_t vrte_cuda_plan_run(vrte_cuda_plan* pl, int32_t iters, double* seconds,
                           vrte_cuda_result* result) {
    return guarded(result, [&]() -> int32_t {
        if (!pl || iters < 1) throw std::invalid_argument("bad plan or iteration count");
        if (pl->device >= 0) VRTE_CUDA_CHECK(cudaSetDevice(pl->device));
        cudaEvent_t a, b;
        VRTE_CUDA_CHECK(cudaEventCreate(&a));
        VRTE_CUDA_CHECK(cudaEventCreate(&b));
        VRTE_CUDA_CHECK(cudaEventRecord(a, pl->st));
        for (int it = 0; it < iters; ++it) run_pipeline(*pl, pl->full_orders);
        VRTE_CUDA_CHECK(cudaEventRecord(b, pl->st));
        VRTE_CUDA_CHECK(cudaEventSynchronize(b));
        float ms = 0;
        VRTE_CUDA_CHECK(cudaEventElapsedTime(&ms, a, b));
        cudaEventDestroy(a);
        cudaEventDestroy(b);
        if (seconds) *seconds = ms * 1e-3 / iters;
        boundary_fallback(*pl, pl->full_orders);
        return finish(*pl, result);
    });
}

int32_t vrte_cuda_plan_fetch(vrte_cuda_plan* pl, double* table) {
    if (!pl || !table) return 5;
    try {
        VRTE_CUDA_CHECK(cudaMemcpyAsync(table, pl->out.p, sizeof(double) * pl->out.n,
                                        cudaMemcpyDeviceToHost, pl->st));
        VRTE_CUDA_CHECK(cudaStreamSynchronize(pl->st));
    } catch (const std::exception&) {
        return 3;
    }
    return 0;
}

int32_t vrte_cuda_plan_fetch_up(vrte_cuda_plan* pl, double* up) {
    if (!pl || !up) return 5;
    try {
        VRTE_CUDA_CHECK(cudaMemcpyAsync(up, pl->up.p, sizeof(double) * pl->up.n,
                                        cudaMemcpyDeviceToHost, pl->st));
        VRTE_CUDA_CHECK(cudaStreamSynchronize(pl->st));
    } catch (const std::exception&) {
        return 3;
    }
    return 0;
}

int32_t vrte_cuda_plan_up_device(vrte_cuda_plan* pl, double** up, size_t* count) {
    if (!pl || !up || !count) return 5;
    *up = pl->up.p;
    *count = pl->up.n;
    return 0;
}

int32_t vrte_cuda_plan_synthesize_device(vrte_cuda_plan* pl, const double* up_all, double* table,
                                         vrte_cuda_result* result) {
    return guarded(result, [&]() -> int32_t {
        if (!pl || !up_all) throw std::invalid_argument("null plan or stacks");
        if (pl->device >= 0) VRTE_CUDA_CHECK(cudaSetDevice(pl->device));
        cudaStream_t st = pl->st;
        const int L = pl->L;
        std::vector<int> slot(L);
        for (int m = 0; m < L; ++m) slot[m] = m;
        pl->slot_all.upload(slot.data(), L, st);
        VRTE_CUDA_CHECK(cudaMemsetAsync(pl->status, 0, sizeof(DeviceStatus), st));
        SynthArgs sa{};
        sa.N = pl->N;
        sa.L = L;
        sa.n_in = pl->n_in;
        sa.n_dphi = pl->n_dphi;
        sa.up = up_all;
        sa.slot_of_order = pl->slot_all.p;
        sa.trig = pl->trig.p;
        sa.post = pl->post.p;
        sa.out = pl->out.p;
        sa.status = pl->status;
        sa.pre = pl->pd.refl_top ? pl->pre.p : nullptr;
        sa.out_lo = pl->out_lo;
        launch_synth(sa, st);
        if (table)
            VRTE_CUDA_CHECK(cudaMemcpyAsync(table, pl->out.p, sizeof(double) * pl->out.n, cudaMemcpyDeviceToHost, st));
        DeviceStatus s{};
        VRTE_CUDA_CHECK(cudaMemcpyAsync(&s, pl->status, sizeof s, cudaMemcpyDeviceToHost, st));
        VRTE_CUDA_CHECK(cudaStreamSynchronize(st));
        if (result) {
            result->clamped = s.clamped;
            result->kernel_launches = 1;
        }
        if (s.code == kFailNegativeIntensity && s.neg_key != 0) {
            const unsigned long long idx = ~s.neg_key;
            VRTE_CUDA_CHECK(cudaMemcpy(&s.value, pl->out.p + idx * 16, sizeof(double), cudaMemcpyDeviceToHost));
        }
        if (s.code != 0) {
            fill_message(result, 3, describe_failure(s, {}, 0, {}));
            return 3;
        }
        if (result) {
            result->status = 0;
            result->message[0] = 0;
        }
        return 0;
    });
}

int32_t vrte_cuda_plan_fetch_modes(vrte_cuda_plan* pl, double* wr, double* wi, double* residual,
                                   double* nu) {
    if (!pl) return 5;
    try {
        const size_t n = (size_t)pl->B * pl->d;
        if (wr)
            VRTE_CUDA_CHECK(cudaMemcpyAsync(wr, pl->wr.p, n * 8, cudaMemcpyDeviceToHost, pl->st));
        if (wi)
            VRTE_CUDA_CHECK(cudaMemcpyAsync(wi, pl->wi.p, n * 8, cudaMemcpyDeviceToHost, pl->st));
        if (residual)
            VRTE_CUDA_CHECK(cudaMemcpyAsync(residual, pl->residual.p, n * 8, cudaMemcpyDeviceToHost, pl->st));
        if (nu)
            VRTE_CUDA_CHECK(cudaMemcpyAsync(nu, pl->nu.p, 2 * n * 8, cudaMemcpyDeviceToHost, pl->st));
        VRTE_CUDA_CHECK(cudaStreamSynchronize(pl->st));
    } catch (const std::exception&) {
        return 3;
    }
    return 0;
}

int32_t vrte_cuda_plan_fetch_ef(vrte_cuda_plan* pl, double* E, double* F) {
    if (!pl) return 5;
    try {
        const size_t n = (size_t)pl->B * pl->d * pl->d;
        if (E) VRTE_CUDA_CHECK(cudaMemcpyAsync(E, pl->E.p, n * 8, cudaMemcpyDeviceToHost, pl->st));
        if (F) VRTE_CUDA_CHECK(cudaMemcpyAsync(F, pl->F.p, n * 8, cudaMemcpyDeviceToHost, pl->st));
        VRTE_CUDA_CHECK(cudaStreamSynchronize(pl->st));
    } catch (const std::exception&) {
        return 3;
    }
    return 0;
}

void vrte_cuda_plan_destroy(vrte_cuda_plan* pl) { delete pl; }

namespace {
// Order-sharded solve over several devices: shard k runs the
// orders m = k, k + D, ... on devices[k] (one host thread each: the pipeline
// has host synchronisation points), the root (shard 0) gathers every shard's
// tau = 0 stacks with peer copies and runs the synthesis over m = 0..L-1.
int32_t brdf_sharded(const vrte_cuda_problem* problem, double* table, vrte_cuda_result* result) {
    const int L = problem->L;
    const int D = std::min(problem->n_devices, L);
    std::vector<std::unique_ptr<PlanLease>> leases(D);
    std::vector<vrte_cuda_result> res(D);
    std::vector<int> rc(D, 0), count(D), offset(D);
    std::vector<std::string> err(D);
    for (int k = 0, off = 0; k < D; ++k) {
        count[k] = (L - k + D - 1) / D;
        offset[k] = off;
        off += count[k];
    }
    auto shard = [&](int k) {
        try {
            vrte_cuda_problem pk = *problem;
            pk.device = problem->devices[k];
            pk.m_begin = k;
            pk.m_stride = D;
            pk.n_orders = count[k];
            pk.n_devices = 1;
            leases[k] = std::make_unique<PlanLease>(pk.device);
            vrte_cuda_plan& pl = **leases[k];
            setup_plan(pl, &pk);
            pl.full_solution = false;
            pl.launches = run_pipeline(pl, false);
            boundary_fallback(pl, false);
            res[k] = vrte_cuda_result{};
            rc[k] = finish(pl, &res[k]);
        } catch (const std::invalid_argument& e) {
            rc[k] = 5;
            err[k] = e.what();
        } catch (const std::exception& e) {
            rc[k] = 3;
            err[k] = e.what();
        }
    };
    {
        std::vector<std::thread> th;
        for (int k = 1; k < D; ++k) th.emplace_back(shard, k);
        shard(0);
        for (auto& t : th) t.join();
    }
    for (int k = 0; k < D; ++k)
        if (rc[k] != 0) {
            if (!err[k].empty()) fill_message(result, rc[k], err[k]);
            else if (result) *result = res[k];
            return rc[k];
        }
    vrte_cuda_plan& root = **leases[0];
    VRTE_CUDA_CHECK(cudaSetDevice(root.device));
    cudaStream_t st = root.st;
    const size_t per = (size_t)root.R * root.d;  // one order's stacks
    root.up_all.alloc((size_t)L * per);
    for (int k = 0; k < D; ++k) {
        const vrte_cuda_plan& pk = **leases[k];
        VRTE_CUDA_CHECK(cudaMemcpyPeerAsync(root.up_all.p + offset[k] * per, root.device, pk.up.p, pk.device,
                                            sizeof(double) * count[k] * per, st));
    }
    std::vector<int> slot(L);
    for (int m = 0; m < L; ++m) slot[m] = offset[m % D] + m / D;
    root.slot_all.upload(slot.data(), L, st);
    VRTE_CUDA_CHECK(cudaMemsetAsync(root.status, 0, sizeof(DeviceStatus), st));
    SynthArgs sa{};
    sa.N = root.N;
    sa.L = L;
    sa.n_in = root.n_in;
    sa.n_dphi = root.n_dphi;
    sa.up = root.up_all.p;
    sa.slot_of_order = root.slot_all.p;
    sa.trig = root.trig.p;
    sa.post = root.post.p;
    sa.out = root.out.p;
    sa.status = root.status;
    sa.pre = root.pd.refl_top ? root.pre.p : nullptr;
    sa.out_lo = root.out_lo;
    launch_synth(sa, st);
    VRTE_CUDA_CHECK(cudaMemcpyAsync(table, root.out.p, sizeof(double) * root.out.n, cudaMemcpyDeviceToHost, st));
    DeviceStatus s{};
    VRTE_CUDA_CHECK(cudaMemcpyAsync(&s, root.status, sizeof s, cudaMemcpyDeviceToHost, st));
    VRTE_CUDA_CHECK(cudaStreamSynchronize(st));
    if (result) {  // stage times: the slowest shard; counters and maxima over the shards
        vrte_cuda_result r = res[0];
        for (int k = 1; k < D; ++k) {
            const vrte_cuda_result& q = res[k];
            for (double vrte_cuda_result::*f :
                 {&vrte_cuda_result::t_homogeneous, &vrte_cuda_result::t_particular, &vrte_cuda_result::t_boundary,
                  &vrte_cuda_result::t_device, &vrte_cuda_result::t_hessenberg, &vrte_cuda_result::t_hqr,
                  &vrte_cuda_result::t_trevc, &vrte_cuda_result::t_refine, &vrte_cuda_result::t_lu_factor,
                  &vrte_cuda_result::t_lu_solve, &vrte_cuda_result::max_eigen_residual,
                  &vrte_cuda_result::max_particular_residual, &vrte_cuda_result::max_balance_residual,
                  &vrte_cuda_result::max_boundary_residual, &vrte_cuda_result::max_boundary_condition})
                r.*f = std::max(r.*f, q.*f);
            for (uint64_t vrte_cuda_result::*f :
                 {&vrte_cuda_result::dithered, &vrte_cuda_result::polished, &vrte_cuda_result::kernel_launches,
                  &vrte_cuda_result::qr_sweeps, &vrte_cuda_result::qr_steps, &vrte_cuda_result::boundary_refined,
                  &vrte_cuda_result::boundary_cond_warnings, &vrte_cuda_result::eigen_slots,
                  &vrte_cuda_result::boundary_fallback, &vrte_cuda_result::particular_extra_steps,
                  &vrte_cuda_result::slots})
                r.*f += q.*f;
        }
        r.clamped = s.clamped;
        r.kernel_launches += 1;
        *result = r;
    }
    if (s.code == kFailNegativeIntensity && s.neg_key != 0) {
        const unsigned long long idx = ~s.neg_key;
        VRTE_CUDA_CHECK(cudaMemcpy(&s.value, root.out.p + idx * 16, sizeof(double), cudaMemcpyDeviceToHost));
    }
    if (s.code != 0) {
        fill_message(result, 3, describe_failure(s, {}, 0, {}));
        return 3;
    }
    if (result) {
        result->status = 0;
        result->message[0] = 0;
    }
    return 0;
}
}  // namespace

int32_t vrte_cuda_brdf(const vrte_cuda_problem* problem, double* table, vrte_cuda_result* result) {
    return guarded(result, [&]() -> int32_t {
        if (!table) throw std::invalid_argument("null table");
        if (problem && problem->n_devices > 1 && problem->devices && problem->n_orders <= 0)
            return brdf_sharded(problem, table, result);
        // A leased plan (device buffers + stream): the entry point is reentrant
        // (vrte.h "every entry point is reentrant") and concurrent callers run
        // concurrently on their own streams; shape changes reallocate.
        if (!problem) throw std::invalid_argument("null problem");
        PlanLease lease(problem->device);
        vrte_cuda_plan& pl = *lease;
        setup_plan(pl, problem);
        pl.full_solution = false;
        pl.launches = run_pipeline(pl, true);
        VRTE_CUDA_CHECK(cudaMemcpyAsync(table, pl.out.p, sizeof(double) * pl.out.n,
                                        cudaMemcpyDeviceToHost, pl.st));
        if (boundary_fallback(pl, true))
            VRTE_CUDA_CHECK(cudaMemcpyAsync(table, pl.out.p, sizeof(double) * pl.out.n,
                                            cudaMemcpyDeviceToHost, pl.st));
        return finish(pl, result);
    });
}

int32_t vrte_cuda_radiance_field(const vrte_cuda_problem* problem, const vrte_cuda_radiance* rad, double* values,
                                 double* reflectance, vrte_cuda_result* result) {
    return guarded(result, [&]() -> int32_t {
        if (!problem || !rad || !values || !reflectance) throw std::invalid_argument("null buffer");
        if (problem->n_in != 1) throw std::invalid_argument("vrte_cuda: the radiance path solves one beam");
        if (rad->n_tau < 1 || rad->n_mu < 1 || rad->n_phi < 1 || !rad->taus || !rad->mus || !rad->phis)
            throw std::invalid_argument("vrte_cuda: empty radiance grid");
        PlanLease lease(problem->device);
        vrte_cuda_plan& pl = *lease;
        setup_plan(pl, problem);
        pl.full_solution = true;
        pl.launches = run_pipeline(pl, false);
        const int code = finish(pl, result);
        if (code != 0) return code;
        // ---- source-function reconstruction (radiance.cu)
        cudaStream_t st = pl.st;
        const int N = pl.N, d = pl.d, P = pl.P, NO = pl.NO, B = pl.B, nmu = rad->n_mu;
        const size_t ld = 4 * (size_t)nmu;
        const double mu0 = problem->mu_in[0];
        std::vector<double> tau_top(P, 0.0), beam_top(P);
        for (int q = 1; q < P; ++q) tau_top[q] = tau_top[q - 1] + problem->tau[q - 1];
        for (int q = 0; q < P; ++q) beam_top[q] = std::exp(-tau_top[q] / mu0);
        auto& rb = pl.rad;
        auto &taus = rb.taus, &mus = rb.mus, &phis = rb.phis, &dtop = rb.dtop, &dbeam = rb.dbeam, &gsf_o = rb.gsf_o;
        auto &wp = rb.wp, &wm = rb.wm, &bb = rb.bb, &acc_a = rb.acc_a, &acc_b = rb.acc_b, &bsrc = rb.bsrc;
        auto &bout = rb.bout, &bbeam = rb.bbeam, &down = rb.down, &bval = rb.bval, &comp = rb.comp;
        auto &field = rb.field, &refl = rb.refl;
        taus.upload(rad->taus, rad->n_tau, st);
        mus.upload(rad->mus, nmu, st);
        phis.upload(rad->phis, rad->n_phi, st);
        dtop.upload(tau_top.data(), P, st);
        dbeam.upload(beam_top.data(), P, st);
        gsf_o.alloc((size_t)pl.L * pl.Lc * 3 * nmu);
        for (auto* b : {&wp, &wm, &acc_a, &acc_b}) b->alloc((size_t)B * ld * d);
        bb.alloc((size_t)B * nmu * 16);
        bsrc.alloc((size_t)P * NO * nmu * 16);
        comp.alloc((size_t)NO * 16 * rad->n_tau * nmu);
        field.alloc((size_t)rad->n_tau * nmu * rad->n_phi * 4);
        refl.alloc(4);
        RadArgs a{};
        a.p = pl.pd;
        a.R = pl.R;
        a.n_tau = rad->n_tau;
        a.n_mu = nmu;
        a.n_phi = rad->n_phi;
        a.mu0 = mu0;
        a.phi0 = rad->phi0;
        a.tau_total = tau_top[P - 1] + problem->tau[P - 1];
        for (int c = 0; c < 4; ++c) a.stokes[c] = rad->stokes[c];
        a.taus = taus.p;
        a.mus = mus.p;
        a.phis = phis.p;
        a.tau_top = dtop.p;
        a.beam_top = dbeam.p;
        a.gsf_n = pl.gsf_n.p;
        a.gsf_b = pl.gsf_b.p;
        a.gsf_o = gsf_o.p;
        a.wp = wp.p;
        a.wm = wm.p;
        a.bb = bb.p;
        a.acc_a = acc_a.p;
        a.acc_b = acc_b.p;
        a.beam_src = bsrc.p;
        a.psi_p = pl.psi_p.p;
        a.psi_m = pl.psi_m.p;
        a.nu = pl.nu.p;
        a.wi = pl.wi.p;
        a.zp = pl.zp.p;
        a.zm = pl.zm.p;
        a.rhs_x = pl.rhs_x.p;
        a.comp = comp.p;
        a.field = field.p;
        a.up = pl.up.p;
        a.refl = refl.p;
        down.alloc(4 * (size_t)d + 4 * (size_t)N);  // base-term stack + reflectance partials
        a.down_bot = down.p;
        a.slot0 = -1;
        for (int mo = 0; mo < NO; ++mo)
            if (pl.m_begin + mo * pl.m_stride == 0) a.slot0 = mo;
        if (problem->base_type != 0 && a.slot0 >= 0) {
            if (!rad->base_out || !rad->base_beam) throw std::invalid_argument("vrte_cuda: missing base rows");
            bout.upload(rad->base_out, (size_t)nmu * N * 16, st);
            bbeam.upload(rad->base_beam, (size_t)nmu * 16, st);
            bval.alloc(16 * (size_t)nmu);
            a.base_out = bout.p;
            a.base_beam = bbeam.p;
            a.base_val = bval.p;
        }
        pl.launches += launch_radiance(a, st);
        VRTE_CUDA_CHECK(cudaMemcpyAsync(values, field.p, sizeof(double) * field.n, cudaMemcpyDeviceToHost, st));
        VRTE_CUDA_CHECK(cudaMemcpyAsync(reflectance, refl.p, sizeof(double) * 4, cudaMemcpyDeviceToHost, st));
        VRTE_CUDA_CHECK(cudaStreamSynchronize(st));
        if (result) result->kernel_launches = pl.launches;
        return 0;
    });
}

int32_t vrte_cuda_synthesize(const vrte_cuda_problem* problem, const double* up, double* table,
                             vrte_cuda_result* result) {
    return guarded(result, [&]() -> int32_t {
        check_problem(problem);
        if (!up || !table) throw std::invalid_argument("null buffer");
        if (problem->device >= 0) VRTE_CUDA_CHECK(cudaSetDevice(problem->device));
        cudaStream_t st;
        VRTE_CUDA_CHECK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
        const int N = problem->N, L = problem->L, n_in = problem->n_in, np = problem->n_dphi;
        const size_t upn = (size_t)L * 4 * n_in * 4 * N;
        DevBuf<double> dup, dtrig, dpost, dout, dpre;
        DevBuf<int> dslot;
        DevBuf<DeviceStatus> dst;
        std::vector<int> slot(L);
        for (int m = 0; m < L; ++m) slot[m] = m;
        dup.upload(up, upn, st);
        dtrig.upload(problem->trig, (size_t)L * np * 2, st);
        dpost.upload(problem->post, (size_t)n_in * 16, st);
        dslot.upload(slot.data(), L, st);
        const int out_lo = problem->refl_top ? problem->out_lo : 0;
        if (problem->refl_top) dpre.upload(problem->pre, (size_t)N * 16, st);
        dout.alloc((size_t)n_in * (N - out_lo) * np * 16);
        dst.alloc(1);
        VRTE_CUDA_CHECK(cudaMemsetAsync(dst.p, 0, sizeof(DeviceStatus), st));
        SynthArgs sa{};
        sa.N = N;
        sa.L = L;
        sa.n_in = n_in;
        sa.n_dphi = np;
        sa.up = dup.p;
        sa.slot_of_order = dslot.p;
        sa.trig = dtrig.p;
        sa.post = dpost.p;
        sa.pre = problem->refl_top ? dpre.p : nullptr;
        sa.out_lo = out_lo;
        sa.out = dout.p;
        sa.status = dst.p;
        launch_synth(sa, st);
        VRTE_CUDA_CHECK(cudaMemcpyAsync(table, dout.p, sizeof(double) * dout.n,
                                        cudaMemcpyDeviceToHost, st));
        DeviceStatus s{};
        VRTE_CUDA_CHECK(cudaMemcpyAsync(&s, dst.p, sizeof s, cudaMemcpyDeviceToHost, st));
        VRTE_CUDA_CHECK(cudaStreamSynchronize(st));
        cudaStreamDestroy(st);
        if (result) {
            result->clamped = s.clamped;
            result->kernel_launches = 1;
        }
        if (s.code == kFailNegativeIntensity && s.neg_key != 0) {
            const unsigned long long idx = ~s.neg_key;
            VRTE_CUDA_CHECK(cudaMemcpy(&s.value, dout.p + idx * 16, sizeof(double), cudaMemcpyDeviceToHost));
        }
        if (s.code != 0) {
            fill_message(result, 3, describe_failure(s, {}, 0, {}));
            return 3;
        }
        if (result) result->status = 0;
        return 0;
    });
}

int32_t vrte_cuda_lu_solve(const double* A, int32_t G, int32_t batch, const double* B, int32_t ncol,
                           double* X, int32_t device) {
    if (!A || !B || !X || G < 1 || batch < 1 || ncol < 1) return 5;
    try {
        if (device >= 0) VRTE_CUDA_CHECK(cudaSetDevice(device));
        cudaStream_t st;
        VRTE_CUDA_CHECK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
        DevBuf<double> dA, dB, dX;
        DevBuf<int> ipiv, perm;
        DevBuf<DeviceStatus> dst;
        dA.upload(A, (size_t)batch * G * G, st);
        dB.upload(B, (size_t)batch * G * ncol, st);
        dX.alloc((size_t)batch * G * ncol);
        ipiv.alloc((size_t)batch * G);
        perm.alloc((size_t)batch * G);
        dst.alloc(1);
        VRTE_CUDA_CHECK(cudaMemsetAsync(dst.p, 0, sizeof(DeviceStatus), st));
        lu_factor_rm(dA.p, G, batch, ipiv.p, perm.p, dst.p, nullptr, st);
        lu_solve_rm(dA.p, G, batch, perm.p, dB.p, dX.p, ncol, st);
        VRTE_CUDA_CHECK(cudaMemcpyAsync(X, dX.p, sizeof(double) * dX.n, cudaMemcpyDeviceToHost, st));
        DeviceStatus s{};
        VRTE_CUDA_CHECK(cudaMemcpyAsync(&s, dst.p, sizeof s, cudaMemcpyDeviceToHost, st));
        VRTE_CUDA_CHECK(cudaStreamSynchronize(st));
        cudaStreamDestroy(st);
        return s.code != 0 ? 3 : 0;
    } catch (const std::exception&) {
        return 3;
    }
}

int32_t vrte_cuda_lu_factor(double* A, int32_t G, int32_t ncols, int32_t batch, int32_t lookahead, int32_t* perm_out,
                            int32_t device) {
    if (!A || !perm_out || G < 1 || ncols < G || batch < 1) return 5;
    try {
        if (device >= 0) VRTE_CUDA_CHECK(cudaSetDevice(device));
        cudaStream_t st;
        VRTE_CUDA_CHECK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
        LuLookahead la;
        int lo_prio = 0, hi_prio = 0;
        VRTE_CUDA_CHECK(cudaDeviceGetStreamPriorityRange(&lo_prio, &hi_prio));
        VRTE_CUDA_CHECK(cudaStreamCreateWithPriority(&la.hi, cudaStreamNonBlocking, hi_prio));
        VRTE_CUDA_CHECK(cudaStreamCreateWithPriority(&la.lo, cudaStreamNonBlocking, lo_prio));
        for (auto& e : la.ev) VRTE_CUDA_CHECK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        DevBuf<double> dA;
        DevBuf<int> ipiv, perm, snap;
        DevBuf<DeviceStatus> dst;
        dA.upload(A, (size_t)batch * G * ncols, st);
        ipiv.alloc((size_t)batch * G);
        perm.alloc((size_t)batch * G);
        snap.alloc((size_t)batch * G);
        la.snap = snap.p;
        dst.alloc(1);
        VRTE_CUDA_CHECK(cudaMemsetAsync(dst.p, 0, sizeof(DeviceStatus), st));
        // bit 1: the columns past G deferred (factor the matrix alone, then
        // lu_rhs_forward on another stream through the per-block snapshots)
        const bool deferred = (lookahead & 2) != 0 && ncols > G;
        LuRhsDefer rd;
        DevBuf<int> rsnap;
        std::vector<cudaEvent_t> rev;
        cudaStream_t s3 = nullptr;
        if (deferred) {
            rd.nblocks = lu_outer_blocks(G);
            rsnap.alloc((size_t)rd.nblocks * batch * G);
            rd.snaps = rsnap.p;
            rev.resize(rd.nblocks);
            for (auto& e : rev) VRTE_CUDA_CHECK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            rd.ev = rev.data();
            VRTE_CUDA_CHECK(cudaStreamCreateWithFlags(&s3, cudaStreamNonBlocking));
        }
        lu_factor_rm(dA.p, G, batch, ipiv.p, perm.p, dst.p, nullptr, st, 0, 0, ncols, deferred ? G : ncols, nullptr,
                     (lookahead & 1) ? &la : nullptr, deferred ? &rd : nullptr);
        if (deferred) {
            lu_rhs_forward(dA.p, G, ncols, ncols - G, batch, rd, 0, 0, s3);
            cudaEvent_t done;
            VRTE_CUDA_CHECK(cudaEventCreateWithFlags(&done, cudaEventDisableTiming));
            VRTE_CUDA_CHECK(cudaEventRecord(done, s3));
            VRTE_CUDA_CHECK(cudaStreamWaitEvent(st, done, 0));
            VRTE_CUDA_CHECK(cudaStreamSynchronize(st));
            cudaEventDestroy(done);
            for (auto& e : rev) cudaEventDestroy(e);
            cudaStreamDestroy(s3);
        }
        VRTE_CUDA_CHECK(cudaMemcpyAsync(A, dA.p, sizeof(double) * dA.n, cudaMemcpyDeviceToHost, st));
        VRTE_CUDA_CHECK(cudaMemcpyAsync(perm_out, perm.p, sizeof(int) * perm.n, cudaMemcpyDeviceToHost, st));
        DeviceStatus s{};
        VRTE_CUDA_CHECK(cudaMemcpyAsync(&s, dst.p, sizeof s, cudaMemcpyDeviceToHost, st));
        VRTE_CUDA_CHECK(cudaStreamSynchronize(st));
        for (auto& e : la.ev) cudaEventDestroy(e);
        cudaStreamDestroy(la.hi);
        cudaStreamDestroy(la.lo);
        cudaStreamDestroy(st);
        return s.code != 0 ? 3 : 0;
    } catch (const std::exception&) {
        return 3;
    }
}

int32_t vrte_cuda_hessenberg(const double* A, int32_t d, int32_t batch, double* H, double* Q,
                             int32_t blocked, int32_t device) {
    if (!A || !H || !Q || d < 1 || batch < 1) return 5;
    try {
        if (device >= 0) VRTE_CUDA_CHECK(cudaSetDevice(device));
        cudaStream_t st;
        VRTE_CUDA_CHECK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
        const size_t n = (size_t)batch * d * d;
        DevBuf<double> dA, dQ, work;
        dA.upload(A, n, st);
        dQ.alloc(n);
        work.alloc((size_t)batch * hessenberg_work_doubles(d));
        if (blocked)
            launch_hessenberg_blocked(dA.p, dQ.p, work.p, d, batch, st);
        else
            launch_hessenberg(dA.p, dQ.p, d, batch, st);
        VRTE_CUDA_CHECK(cudaMemcpyAsync(H, dA.p, sizeof(double) * n, cudaMemcpyDeviceToHost, st));
        VRTE_CUDA_CHECK(cudaMemcpyAsync(Q, dQ.p, sizeof(double) * n, cudaMemcpyDeviceToHost, st));
        VRTE_CUDA_CHECK(cudaStreamSynchronize(st));
        cudaStreamDestroy(st);
        return 0;
    } catch (const std::exception&) {
        return 3;
    }
}

int32_t vrte_cuda_schur(const double* A, int32_t d, int32_t batch, double* T, double* Z, double* wr,
                        double* wi, int32_t device) {
    return vrte_cuda_schur_trace(A, d, batch, T, Z, wr, wi, device, nullptr, nullptr);
}

int32_t vrte_cuda_schur_trace(const double* A, int32_t d, int32_t batch, double* T, double* Z, double* wr,
                              double* wi, int32_t device, double* trace, double* qr_ms) {
    if (!A || !T || !Z || !wr || !wi || d < 1 || batch < 1) return 5;
    try {
        if (device >= 0) VRTE_CUDA_CHECK(cudaSetDevice(device));
        cudaStream_t st;
        VRTE_CUDA_CHECK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
        const size_t n = (size_t)batch * d * d;
        DevBuf<double> dA, dZ, work, dwr, dwi;
        DevBuf<DeviceStatus> dst;
        dA.upload(A, n, st);
        dZ.alloc(n);
        dwr.alloc((size_t)batch * d);
        dwi.alloc((size_t)batch * d);
        dst.alloc(1);
        VRTE_CUDA_CHECK(cudaMemsetAsync(dst.p, 0, sizeof(DeviceStatus), st));
        work.alloc((size_t)batch * hessenberg_work_doubles(d));
        launch_hessenberg_blocked(dA.p, dZ.p, work.p, d, batch, st);
        cudaEvent_t e0, e1;
        VRTE_CUDA_CHECK(cudaEventCreate(&e0));
        VRTE_CUDA_CHECK(cudaEventCreate(&e1));
        VRTE_CUDA_CHECK(cudaEventRecord(e0, st));
        DevBuf<double> dtr;
        if (trace) dtr.alloc((size_t)batch * 8);
        launch_hqr(dA.p, dZ.p, dwr.p, dwi.p, d, batch, dst.p, st, trace ? dtr.p : nullptr);
        VRTE_CUDA_CHECK(cudaEventRecord(e1, st));
        if (trace)
            VRTE_CUDA_CHECK(cudaMemcpyAsync(trace, dtr.p, sizeof(double) * dtr.n, cudaMemcpyDeviceToHost, st));
        VRTE_CUDA_CHECK(cudaMemcpyAsync(T, dA.p, sizeof(double) * n, cudaMemcpyDeviceToHost, st));
        VRTE_CUDA_CHECK(cudaMemcpyAsync(Z, dZ.p, sizeof(double) * n, cudaMemcpyDeviceToHost, st));
        VRTE_CUDA_CHECK(cudaMemcpyAsync(wr, dwr.p, sizeof(double) * batch * d, cudaMemcpyDeviceToHost, st));
        VRTE_CUDA_CHECK(cudaMemcpyAsync(wi, dwi.p, sizeof(double) * batch * d, cudaMemcpyDeviceToHost, st));
        DeviceStatus s{};
        VRTE_CUDA_CHECK(cudaMemcpyAsync(&s, dst.p, sizeof s, cudaMemcpyDeviceToHost, st));
        VRTE_CUDA_CHECK(cudaStreamSynchronize(st));
        cudaStreamDestroy(st);
        if (qr_ms) {
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            *qr_ms = ms;
        }
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        return s.code != 0 ? 3 : 0;
    } catch (const std::exception&) {
        return 3;
    }
}

}  // extern "C"
