// runtime.cu -- the C ABI of libpic.so (include/pic.h): validation,
// workspace carving, the per-step schedule, CUDA graph capture, the z-slab
// exchanges (NCCL or in-process device copies), stage timing and the sticky
// device error word.
//
// Per step n:
//   A  a1   n % K == 0: sort A -> B per species (sort.cu), dropping dead slots
//      a2-6 fused particle kernel per species (input B on a sort step else A,
//           output A in place), deposit into J_cur; [slabs] tail kernel for
//           particles received since the last sort; migration headers
//   X1 [slabs] J ghost planes + migrating particles to ranks r-1, r+1
//   B  [slabs] add received J planes, append received particles;
//      a7   B half (from plane -1 on slabs), E full (+ J fold, zero J_next)
//   X2 [slabs] E ghost planes
//   C  a7   B half
//   X3 [slabs] B ghost planes
//   then swap J_cur / J_next.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include <nccl.h>

#include "../../include/pic.h"
#include "kernels.cuh"

using namespace pic;

namespace {

constexpr size_t kAlign = 256;
inline size_t align_up(size_t v) { return (v + kAlign - 1) / kAlign * kAlign; }
constexpr int64_t kDefaultMigrate = 65536;
constexpr int kAccSlots = 16;   // diagnostics accumulators, see k_diag_nodes

struct Layout {
    GridDev g{};
    int64_t ncells = 0, n_sc = 0;
    int64_t cap[PIC_MAX_SPECIES] = {};
    int64_t cap_max = 0;
    int64_t mig = 0;   // migration capacity (per species and direction), 0 on one rank
    size_t off_eb = 0, off_bh = 0, off_j[2] = {}, off_sp[PIC_MAX_SPECIES][2] = {}, off_scoff[PIC_MAX_SPECIES] = {};
    size_t off_key = 0, off_slot = 0, off_perm_tmp = 0, off_perm = 0, off_count = 0, off_start = 0,
           off_bsums = 0, off_bsums2 = 0, off_err = 0, off_stat = 0, off_n = 0;
    size_t off_msend[PIC_MAX_SPECIES][2] = {}, off_mrecv[PIC_MAX_SPECIES][2] = {}, off_mcnt = 0;
    size_t off_jrecv[2] = {};
    size_t off_rho = 0, off_rho_prev = 0, off_gauss0 = 0, off_acc = 0;   // diagnostics
    size_t off_laser = 0, off_step = 0;                                  // NEXT-1 open z
    size_t off_scale = 0;                                                // J-tile scales
    size_t total = 0;
};

std::string validate(const pic_config *c)
{
    if (!c) return "cfg is NULL";
    if (c->nx <= 0 || c->ny <= 0 || c->nz <= 0) return "grid extents must be positive";
    if (!(c->dx > 0 && c->dy > 0 && c->dz > 0)) return "cell sizes must be positive";
    if (!(c->c > 0) || !(c->dt > 0)) return "c and dt must be positive";
    const double dt_cfl = 1.0 / (c->c * std::sqrt(1.0 / (c->dx * c->dx) + 1.0 / (c->dy * c->dy) +
                                                  1.0 / (c->dz * c->dz)));
    if (c->dt > dt_cfl * (1.0 + 1e-12)) return "CFL violated: dt > 1/(c sqrt(1/dx^2+1/dy^2+1/dz^2))";
    if (c->n_species < 1 || c->n_species > PIC_MAX_SPECIES) return "n_species out of range";
    for (int s = 0; s < c->n_species; ++s) {
        if (!(c->m[s] > 0)) return "species mass must be positive";
        if (c->capacity[s] < 0 || c->capacity[s] >= (int64_t(1) << 31)) return "capacity out of range";
        if (!std::isfinite(c->q[s]) || !std::isfinite(c->w[s])) return "non-finite q or w";
    }
    if (c->nranks < 1 || c->rank < 0 || c->rank >= c->nranks) return "bad rank / nranks";
    if (c->supercell < 1) return "supercell must be >= 1";
    if (c->halo < 0 || c->halo > 2) return "halo must be 1 or 2 (0 = 1)";
    if (c->bc_z != PIC_BC_PERIODIC && c->bc_z != PIC_BC_OPEN) return "bc_z must be PIC_BC_PERIODIC or PIC_BC_OPEN";
    if (c->bc_z == PIC_BC_OPEN && c->nz < 3) return "an open z box needs nz >= 3";
    if (c->bc_z == PIC_BC_OPEN &&
        !(std::isfinite(c->laser_e0) && std::isfinite(c->laser_omega) && c->laser_ramp >= 0.0 &&
          std::isfinite(c->laser_ramp) && std::isfinite(c->laser_t0) && std::isfinite(c->laser_pol[0]) &&
          std::isfinite(c->laser_pol[1])))
        return "bad laser parameters";
    const bool explicit_slab = c->nranks > 1 && (c->slab_lo != 0 || c->slab_hi != 0);
    if (explicit_slab) {
        if (!(c->slab_lo >= 0 && c->slab_lo < c->slab_hi && c->slab_hi <= c->nz)) return "bad slab_lo / slab_hi";
        if ((c->rank == 0) != (c->slab_lo == 0) || (c->rank == c->nranks - 1) != (c->slab_hi == c->nz))
            return "slab_lo / slab_hi: rank 0 starts at 0, the last rank ends at nz";
    } else if (c->nz % c->nranks) {
        return "nz must be divisible by nranks (or set slab_lo / slab_hi)";
    }
    const int64_t nzl = explicit_slab ? c->slab_hi - c->slab_lo : c->nz / c->nranks;
    if (c->nx % c->supercell || c->ny % c->supercell || nzl % c->supercell)
        return "supercell must divide nx, ny and the slab thickness";
    if (c->nranks > 1 && nzl < 4) return "z slabs must be at least 4 cells thick";
    if (c->sort_every < 0) return "sort_every must be >= 0";
    if (c->migrate_capacity < 0 || c->migrate_capacity >= (int64_t(1) << 28)) return "bad migrate_capacity";
    if (c->nx * c->ny * nzl >= (int64_t(1) << 31)) return "local grid too large";
    return "";
}

Layout make_layout(const pic_config *c)
{
    Layout L;
    GridDev &g = L.g;
    g.nx = (int)c->nx;
    g.ny = (int)c->ny;
    const bool explicit_slab = c->nranks > 1 && (c->slab_lo != 0 || c->slab_hi != 0);
    g.nz = (int)(explicit_slab ? c->slab_hi - c->slab_lo : c->nz / c->nranks);
    g.nz_global = (int)c->nz;
    g.k0 = (int)(explicit_slab ? c->slab_lo : c->rank * g.nz);
    g.X = g.nx + 2 * kGhost;
    g.X = (g.X + 3) / 4 * 4;   // 32-byte rows (TMA global strides need 16; tile boxes start 32-byte aligned)
    g.Y = g.ny + 2 * kGhost;
    g.Z = g.nz + 2 * kGhost;
    g.cs = (int64_t)g.X * g.Y * g.Z;
    g.cs += (g.cs & 1);
    g.dx = c->dx; g.dy = c->dy; g.dz = c->dz;
    g.inv_dx = 1.0 / c->dx; g.inv_dy = 1.0 / c->dy; g.inv_dz = 1.0 / c->dz;
    g.dt = c->dt; g.c = c->c;
    g.Lx = c->nx * c->dx; g.Ly = c->ny * c->dy; g.Lz = c->nz * c->dz;
    g.S = (int)c->supercell;
    g.H = c->halo ? (int)c->halo : 1;
    g.nsx = g.nx / g.S; g.nsy = g.ny / g.S; g.nsz = g.nz / g.S;
    g.open_z = c->bc_z == PIC_BC_OPEN;
    g.periodic_z_local = (c->nranks == 1) && !g.open_z;
    g.nranks = (int)c->nranks;
    g.rank = (int)c->rank;
    g.zlo = c->nranks == 1 ? 0.0 : (double)g.k0 * c->dz;
    g.zhi = c->nranks == 1 ? g.Lz : (c->rank == c->nranks - 1 ? g.Lz : (double)(g.k0 + g.nz) * c->dz);
    g.open_lo = g.open_z && c->rank == 0;
    g.open_hi = g.open_z && c->rank == c->nranks - 1;
    g.zmax = g.open_z ? (double)(c->nz - 1) * c->dz : g.Lz;
    g.mur_a = (c->c * c->dt - c->dz) / (c->c * c->dt + c->dz);
    g.laser = nullptr;   // set by pic_init
    L.ncells = (int64_t)g.nx * g.ny * g.nz;
    L.n_sc = (int64_t)g.nsx * g.nsy * g.nsz;
    L.mig = c->nranks > 1 ? (c->migrate_capacity ? c->migrate_capacity : kDefaultMigrate) : 0;
    size_t o = 0;
    L.off_eb = o; o = align_up(o + sizeof(double) * 6 * (size_t)g.cs);
    for (int b = 0; b < 2; ++b) { L.off_j[b] = o; o = align_up(o + sizeof(double) * 3 * (size_t)g.cs); }
    L.off_bh = o; o = align_up(o + sizeof(double) * 3 * (size_t)g.cs);   // B^{n+1/2}
    for (int s = 0; s < c->n_species; ++s) {
        L.cap[s] = c->capacity[s];
        L.cap_max = std::max(L.cap_max, L.cap[s]);
        for (int b = 0; b < 2; ++b) {
            L.off_sp[s][b] = o;
            o = align_up(o + (sizeof(double) * 6 + sizeof(uint64_t)) * (size_t)L.cap[s] + 8 * kAlign);
        }
        L.off_scoff[s] = o; o = align_up(o + sizeof(int64_t) * (size_t)(L.n_sc + 1));
        if (L.mig) {
            for (int d = 0; d < 2; ++d) {
                L.off_msend[s][d] = o; o = align_up(o + sizeof(double) * (size_t)(1 + 7 * L.mig));
                L.off_mrecv[s][d] = o; o = align_up(o + sizeof(double) * (size_t)(1 + 7 * L.mig));
            }
        }
    }
    if (L.mig) {
        for (int d = 0; d < 2; ++d) {
            L.off_jrecv[d] = o;
            o = align_up(o + sizeof(double) * 3 * 2 * (size_t)g.X * g.Y);
        }
    }
    // +1: compact_live scans n + 1 entries (k_live_flags writes flag[n] into
    // perm_tmp, k_scan_add writes perm[n])
    const size_t capm = (size_t)std::max<int64_t>(L.cap_max, 1) + 1;
    L.off_key = o; o = align_up(o + 4 * capm);
    L.off_slot = o; o = align_up(o + 4 * capm);
    L.off_perm_tmp = o; o = align_up(o + 4 * capm);
    L.off_perm = o; o = align_up(o + 4 * capm);
    L.off_count = o; o = align_up(o + 4 * (size_t)(L.ncells + 1));
    L.off_start = o; o = align_up(o + 4 * (size_t)(L.ncells + 1));
    L.off_bsums = o; o = align_up(o + 4 * scan_block_count(L.ncells + 1));
    L.off_bsums2 = o; o = align_up(o + 4 * scan_block_count(L.cap_max + 1));   // compact_live
    L.off_err = o; o = align_up(o + 64);
    L.off_stat = o; o = align_up(o + 2 * PIC_MAX_SPECIES * sizeof(unsigned));
    L.off_n = o; o = align_up(o + PIC_MAX_SPECIES * sizeof(int64_t));
    L.off_mcnt = o; o = align_up(o + 2 * PIC_MAX_SPECIES * sizeof(unsigned));
    L.off_rho = o; o = align_up(o + sizeof(double) * (size_t)g.cs);
    L.off_rho_prev = o; o = align_up(o + sizeof(double) * (size_t)g.cs);
    L.off_gauss0 = o; o = align_up(o + sizeof(double) * (size_t)g.cs);
    L.off_acc = o; o = align_up(o + sizeof(double) * kAccSlots);
    L.off_laser = o; o = align_up(o + sizeof(double) * 8);
    L.off_step = o; o = align_up(o + sizeof(int64_t));
    L.off_scale = o; o = align_up(o + sizeof(double) * 2 * PIC_MAX_SPECIES);
    L.total = o;
    return L;
}

// bytes per SoA column of a particle store (+16: a staged chunk may read
// up to 2 nodes past the last particle)
static size_t particle_col_bytes(int64_t cap) { return align_up(sizeof(double) * (size_t)cap + 16); }

ParticlesDev carve_particles(char *base, size_t off, int64_t cap)
{
    ParticlesDev p;
    const size_t col = particle_col_bytes(cap);
    char *b = base + off;
    p.x = (double *)(b + 0 * col);
    p.y = (double *)(b + 1 * col);
    p.z = (double *)(b + 2 * col);
    p.ux = (double *)(b + 3 * col);
    p.uy = (double *)(b + 4 * col);
    p.uz = (double *)(b + 5 * col);
    p.id = (uint64_t *)(b + 6 * col);
    return p;
}

const char *err_names(int code)
{
    switch (code) {
    case PIC_OK: return "ok";
    case PIC_EINVAL: return "invalid argument or configuration";
    case PIC_ENOMEM: return "workspace too small";
    case PIC_ECAPACITY: return "capacity exceeded";
    case PIC_ESTATE: return "invalid call order";
    case PIC_EDISPLACEMENT: return "a particle moved one cell or more in one step";
    case PIC_ENONFINITE: return "non-finite particle state";
    case PIC_ECUDA: return "CUDA error";
    case PIC_ENCCL: return "NCCL error";
    default: return "unknown error";
    }
}

// ---- NCCL, loaded at run time (only z-slab runs need it): the copy already
// loaded into the process (torch's, when torch.distributed initialised NCCL),
// else $PIC_NCCL_LIB (the Python binding points it at the torch wheel's
// nvidia/nccl/lib/libnccl.so.2), else the loader's libnccl.so.2 ----
struct NcclApi {
    void *h = nullptr;
    ncclResult_t (*getUniqueId)(ncclUniqueId *) = nullptr;
    ncclResult_t (*commInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*send)(const void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*recv)(void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*groupStart)() = nullptr;
    ncclResult_t (*groupEnd)() = nullptr;
    const char *(*errorString)(ncclResult_t) = nullptr;
};

NcclApi *nccl_api()
{
    static NcclApi api;
    static bool tried = false;
    if (tried) return api.h ? &api : nullptr;
    tried = true;
    void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    const char *env = std::getenv("PIC_NCCL_LIB");
    if (!h && env && *env) h = dlopen(env, RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return nullptr;
    api.getUniqueId = (decltype(api.getUniqueId))dlsym(h, "ncclGetUniqueId");
    api.commInitRank = (decltype(api.commInitRank))dlsym(h, "ncclCommInitRank");
    api.commDestroy = (decltype(api.commDestroy))dlsym(h, "ncclCommDestroy");
    api.send = (decltype(api.send))dlsym(h, "ncclSend");
    api.recv = (decltype(api.recv))dlsym(h, "ncclRecv");
    api.groupStart = (decltype(api.groupStart))dlsym(h, "ncclGroupStart");
    api.groupEnd = (decltype(api.groupEnd))dlsym(h, "ncclGroupEnd");
    api.errorString = (decltype(api.errorString))dlsym(h, "ncclGetErrorString");
    if (!api.getUniqueId || !api.commInitRank || !api.send || !api.recv || !api.groupStart ||
        !api.groupEnd || !api.commDestroy)
        return nullptr;
    api.h = h;
    return &api;
}

// one point-to-point message of an exchange: every rank sends `send` toward
// dir (0 = rank-1, 1 = rank+1) and receives the same message of the rank on
// the other side into `recv`
struct Msg {
    double *send;
    double *recv;
    size_t count;
    int dir;
};

}  // namespace

struct pic_ctx {
    pic_config cfg{};
    Layout L;
    char *ws = nullptr;
    cudaStream_t st = nullptr;
    double *EB = nullptr;
    double *Bh = nullptr;      // B^{n+1/2} for the next E update (bit-equal to a half step of EB's B)
    bool bh_stale = false;     // Bh must be recomputed from EB (after pic_set_fields / pic_laser_preload)
    bool prep_ready = false;   // the next step's J-tile scales are prepared (by k_e_full)
    double *J[2] = {nullptr, nullptr};
    int jcur = 0;              // J buffer receiving the next deposit
    int jlast = 1;             // J buffer holding J^{n-1/2}
    ParticlesDev A[PIC_MAX_SPECIES], B[PIC_MAX_SPECIES];
    int64_t *sc_off[PIC_MAX_SPECIES] = {};
    int64_t *dev_n = nullptr;  // [species] particle slots in use (sorted region + tail)
    bool has_particles[PIC_MAX_SPECIES] = {};
    SortScratch sort{};
    unsigned *err = nullptr;
    unsigned *u2max[2] = {nullptr, nullptr};   // [parity][species], see SpeciesDev
    MigrateDev mig[PIC_MAX_SPECIES];
    double *mrecv[PIC_MAX_SPECIES][2] = {};
    double *jrecv[2] = {nullptr, nullptr};     // [from rank-1, from rank+1]
    // diagnostics (diag.cu): padded node arrays and accumulators
    double *rho = nullptr, *rho_prev = nullptr, *gauss0 = nullptr, *acc = nullptr;
    // NEXT-1 open z: incident values of the current step and the device step counter
    double *laser = nullptr;
    int64_t *dev_step = nullptr;
    double *tile_scale = nullptr;   // [species][2] fixed-point J-tile scale of the step
    double laser_par[6] = {0, 0, 0, 0, 0, 0};   // e0, omega, ramp, t0, pol_x, pol_y
    int64_t diag_last_step = -2;
    bool diag_have_g0 = false;
    int64_t step_index = 0;
    bool use_tile = false;     // fused supercell kernel (else the naive kernel)
    bool slabs = false;        // nranks > 1
    bool local_group = false;  // slabs exchanged by pic_step_group (no NCCL)
    bool ghosts_stale = false; // E/B z ghosts need an exchange (after pic_set_fields)
    CUtensorMap eb_map;        // TMA descriptor of the padded E/B array [6][Z][Y][X]
    // Occupied supercell layers (single domain only, `occ_trim`): the particle
    // kernel is launched over the layers holding particles since the last sort
    // (the empty layers' CTAs cost 0.56 ms of a 3.9 ms C5_1g launch).  After a
    // sort, k_occ_range writes the exact range into the mapped pinned h_occ
    // (event ev_occ, polled without waiting); occ holds a range known to
    // contain the occupied layers (push_layers).
    bool occ_trim = false;
    int *d_occ = nullptr;      // device alias of the mapped pinned h_occ
    int *h_occ = nullptr;
    cudaEvent_t ev_occ = nullptr;
    bool occ_pending = false;
    int occ[2] = {0, -1};      // {first, last} (last < first: no particles)
    int push_zr[2] = {0, 0};   // layers [first, end) the steps being enqueued push
    int prev_zr[2] = {0, 0};   // ... and the previous step pushed (J zero at init: none)
    CUtensorMap pmap[PIC_MAX_SPECIES][2];   // TMA descriptors of the particle stores A, B ([6][cap + 2])
    int num_sms = 148;
    ncclComm_t comm = nullptr;
    // z slabs: the J ghost / migration exchange of a step runs on st_x while
    // the interior supercell layers are pushed on st (fork/join by events,
    // captured in the step graph); zb = boundary layers per slab end
    cudaStream_t st_x = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    int zb = 0;
    std::string last_error;
    // graphs keyed by (sort_now, jcur)
    cudaGraphExec_t graph[2][2] = {{nullptr, nullptr}, {nullptr, nullptr}};
    int graph_zr[2][2][4] = {};   // push_zr and prev_zr each graph was captured with
    int graph_launches[2][2] = {{0, 0}, {0, 0}};
    bool graphs_valid = false;
    int64_t launches = 0;
    // profiling
    std::vector<cudaEvent_t> ev_pool;
    size_t ev_used = 0;
    std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> ev_marks;
    double stage_ms[4] = {0, 0, 0, 0};
    int64_t particle_launches = 0;
};

namespace {

int fail(pic_ctx *ctx, int code, const std::string &msg)
{
    if (ctx) ctx->last_error = msg.empty() ? err_names(code) : msg;
    return code;
}

int cuda_fail(pic_ctx *ctx, cudaError_t e, const char *where)
{
    return fail(ctx, PIC_ECUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

#define PIC_CUDA(ctx, call)                                        \
    do {                                                           \
        cudaError_t e_ = (call);                                   \
        if (e_ != cudaSuccess) return cuda_fail((ctx), e_, #call); \
    } while (0)

cudaEvent_t take_event(pic_ctx *ctx)
{
    if (ctx->ev_used == ctx->ev_pool.size()) {
        cudaEvent_t e;
        cudaEventCreate(&e);
        ctx->ev_pool.push_back(e);
    }
    return ctx->ev_pool[ctx->ev_used++];
}

struct StageMark {
    pic_ctx *ctx;
    int stage;
    cudaEvent_t a = nullptr;
    StageMark(pic_ctx *c, int s, bool on) : ctx(c), stage(s)
    {
        if (on) {
            a = take_event(ctx);
            cudaEventRecord(a, ctx->st);
        }
    }
    ~StageMark()
    {
        if (a) {
            cudaEvent_t b = take_event(ctx);
            cudaEventRecord(b, ctx->st);
            ctx->ev_marks.push_back({stage, {a, b}});
        }
    }
};

SpeciesDev species_dev(pic_ctx *ctx, int s, int jcur)
{
    const GridDev &g = ctx->L.g;
    SpeciesDev sp;
    sp.qw = ctx->cfg.q[s] * ctx->cfg.w[s];
    sp.h = ctx->cfg.q[s] * g.dt / (2.0 * ctx->cfg.m[s] * g.c);
    sp.u2max_in = ctx->u2max[jcur] + s;
    sp.u2max_out = ctx->u2max[1 - jcur] + s;
    sp.kx = sp.qw / (g.dt * g.dy * g.dz);
    sp.ky = sp.qw / (g.dt * g.dx * g.dz);
    sp.kz = sp.qw / (g.dt * g.dx * g.dy);
    sp.scale = ctx->tile_scale + 2 * s;
    sp.mig = ctx->mig[s];
    return sp;
}

// ---- exchanges (slabs) ----
size_t plane_pair(const GridDev &g) { return 2 * (size_t)g.X * g.Y; }
// padded-array offset of local plane k (first of the pair) within one component
size_t plane_off(const GridDev &g, int k) { return (size_t)(k + kGhost) * g.X * g.Y; }

std::vector<Msg> msgs_fields(pic_ctx *ctx, int c0, int c1)
{
    // send own boundary planes {0,1} down and {nz-2,nz-1} up; receive into the
    // ghost planes {nz, nz+1} (from rank+1) and {-2,-1} (from rank-1)
    const GridDev &g = ctx->L.g;
    std::vector<Msg> m;
    for (int c = c0; c < c1; ++c) {
        double *F = ctx->EB + c * g.cs;
        m.push_back({F + plane_off(g, 0), F + plane_off(g, g.nz), plane_pair(g), 0});
        m.push_back({F + plane_off(g, g.nz - 2), F + plane_off(g, -2), plane_pair(g), 1});
    }
    return m;
}

std::vector<Msg> msgs_current(pic_ctx *ctx, int jcur)
{
    // own J ghost planes {-2,-1} go down, {nz,nz+1} go up; the neighbours'
    // arrive in jrecv[1] (from rank+1) and jrecv[0] (from rank-1)
    const GridDev &g = ctx->L.g;
    std::vector<Msg> m;
    for (int c = 0; c < 3; ++c) {
        double *Jc = ctx->J[jcur] + c * g.cs;
        m.push_back({Jc + plane_off(g, -2), ctx->jrecv[1] + c * plane_pair(g), plane_pair(g), 0});
        m.push_back({Jc + plane_off(g, g.nz), ctx->jrecv[0] + c * plane_pair(g), plane_pair(g), 1});
    }
    for (int s = 0; s < ctx->cfg.n_species; ++s) {
        const size_t n = 1 + 7 * (size_t)ctx->L.mig;
        m.push_back({ctx->mig[s].send[0], ctx->mrecv[s][1], n, 0});
        m.push_back({ctx->mig[s].send[1], ctx->mrecv[s][0], n, 1});
    }
    return m;
}

// the ring of slabs is cut at an open z box's faces (NEXT-1): rank 0 has no
// lower and the last rank no upper neighbour
bool has_neighbour(const pic_config &c, int rank, int dir)
{
    if (c.bc_z != PIC_BC_OPEN) return true;
    return dir == 0 ? rank > 0 : rank < c.nranks - 1;
}

int exchange_nccl(pic_ctx *ctx, const std::vector<Msg> &msgs, cudaStream_t st = nullptr)
{
    if (!st) st = ctx->st;
    NcclApi *api = nccl_api();
    if (!api || !ctx->comm) return fail(ctx, PIC_ENCCL, "NCCL not initialised");
    const int r = (int)ctx->cfg.rank, n = (int)ctx->cfg.nranks;
    const int dn = (r + n - 1) % n, up = (r + 1) % n;
    const bool has_dn = has_neighbour(ctx->cfg, r, 0), has_up = has_neighbour(ctx->cfg, r, 1);
    ncclResult_t e = api->groupStart();
    // sends and receives are each posted in message order, so with two ranks
    // (dn == up) the i-th send matches the peer's i-th receive; a message of
    // direction d goes to the neighbour on side d and arrives from the other side
    for (const Msg &m : msgs)
        if (e == ncclSuccess && (m.dir == 0 ? has_dn : has_up))
            e = api->send(m.send, m.count, ncclFloat64, m.dir == 0 ? dn : up, ctx->comm, st);
    for (const Msg &m : msgs)
        if (e == ncclSuccess && (m.dir == 0 ? has_up : has_dn))
            e = api->recv(m.recv, m.count, ncclFloat64, m.dir == 0 ? up : dn, ctx->comm, st);
    const ncclResult_t e2 = api->groupEnd();
    if (e != ncclSuccess || e2 != ncclSuccess)
        return fail(ctx, PIC_ENCCL, std::string("NCCL exchange: ") +
                                        (api->errorString ? api->errorString(e != ncclSuccess ? e : e2) : ""));
    return PIC_OK;
}

// copies message i of every rank into its receiver (in-process slab group)
int exchange_local(pic_ctx *const *ctxs, int n, const std::vector<std::vector<Msg>> &msgs)
{
    for (int r = 0; r < n; ++r) {
        for (size_t i = 0; i < msgs[r].size(); ++i) {
            const Msg &m = msgs[r][i];
            if (!has_neighbour(ctxs[r]->cfg, r, m.dir == 0 ? 1 : 0)) continue;   // open face
            const int src = m.dir == 0 ? (r + 1) % n : (r + n - 1) % n;   // who sends toward r
            PIC_CUDA(ctxs[r], cudaMemcpyAsync(m.recv, msgs[src][i].send, m.count * sizeof(double),
                                              cudaMemcpyDeviceToDevice, ctxs[r]->st));
        }
    }
    return PIC_OK;
}

// k_occ_range over the species with particles, written into the mapped
// pinned h_occ (part of a sort step's graph; the event is recorded after the
// launch)
static_assert(kOccMaxSpecies == PIC_MAX_SPECIES, "OccRange holds every species");
void enqueue_occ_range(pic_ctx *ctx)
{
    OccRange a{};
    for (int s = 0; s < ctx->cfg.n_species; ++s)
        if (ctx->has_particles[s]) a.sc_off[a.ns++] = ctx->sc_off[s];
    a.per_layer = (int64_t)ctx->L.g.nsx * ctx->L.g.nsy;
    a.nsz = ctx->L.g.nsz;
    launch_occ_range(a, ctx->d_occ, ctx->st);   // straight into the mapped pinned h_occ
}

// the exact occupied range of the last sort once its copy has landed
// (polled: never waits, so the host keeps enqueueing ahead of the device)
int poll_occ(pic_ctx *ctx, bool wait)
{
    if (!ctx->occ_pending) return PIC_OK;
    if (wait) {
        PIC_CUDA(ctx, cudaEventSynchronize(ctx->ev_occ));
    } else {
        const cudaError_t e = cudaEventQuery(ctx->ev_occ);
        if (e == cudaErrorNotReady) return PIC_OK;
        if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaEventQuery");
    }
    ctx->occ[0] = ctx->h_occ[0];
    ctx->occ[1] = ctx->h_occ[1];
    if (ctx->occ[0] < 0) ctx->occ[1] = -1;   // none
    ctx->occ_pending = false;
    return PIC_OK;
}

// The supercell layers [first, end) the particle kernel of a step pushes.
// Between sorts every particle stays in its sorted supercell's range, so a
// range holding the occupied layers of the last sort is right: the exact
// one once its copy has landed, else the one that step pushed.  A step that
// sorts first pushes that range widened by the farthest a particle can have
// moved since the last sort (less than one cell per step by the CFL
// condition, at most K steps: ceil(K / S) + 1 layers; the whole box when
// that reaches a periodic z end), and that widened range stands for the new
// sort's until its exact one lands.
void push_layers(pic_ctx *ctx, bool sort_now, int zr[2])
{
    const int nsz = ctx->L.g.nsz;
    zr[0] = 0;
    zr[1] = nsz;
    if (!ctx->occ_trim) return;
    int lo = ctx->occ[0], hi = ctx->occ[1];
    if (hi >= lo && sort_now) {
        const int64_t S = ctx->cfg.supercell, K = std::max<int64_t>(ctx->cfg.sort_every, 1);
        const int m = (int)((K + S - 1) / S) + 1;
        lo -= m;
        hi += m;
        if (ctx->L.g.periodic_z_local && (lo < 0 || hi >= nsz)) {
            lo = 0;
            hi = nsz - 1;
        }
        lo = std::max(lo, 0);
        hi = std::min(hi, nsz - 1);
        ctx->occ[0] = lo;
        ctx->occ[1] = hi;
    }
    if (hi < lo) {   // no particles
        zr[1] = 0;
        return;
    }
    zr[0] = lo;
    zr[1] = hi + 1;
}

// The padded J planes [lo, hi] the particle kernel of a step pushing the
// supercell layers zr = [first, end) can deposit into: the J tiles of those
// layers, S (z0 - 1) - H - 1 + ... (TileGeom: S + 2H + 3 planes from
// S z - H - 1), widened for the particles on the global path, which have
// drifted beyond their tile since the last sort (less than one cell per step,
// at most K steps; 2 more for the edges of a path); the whole array when
// that reaches a periodic z end, when there is no sort, or when the layers
// are not tracked (lo > hi: none).
void j_planes(const pic_ctx *ctx, const int zr[2], int &lo, int &hi)
{
    const GridDev &g = ctx->L.g;
    lo = 0;
    hi = g.Z - 1;
    const int64_t K = ctx->cfg.sort_every;
    if (!ctx->occ_trim || K <= 0) return;
    if (zr[1] <= zr[0]) {
        lo = 1;
        hi = 0;
        return;
    }
    const int S = g.S, H = g.H, m = (int)std::min<int64_t>(K + 2, g.Z);
    int a = zr[0] * S - H - 1 + kGhost - m, b = (zr[1] - 1) * S - H - 1 + kGhost + (S + 2 * H + 3) - 1 + m;
    if (g.periodic_z_local && (a < kGhost || b >= g.nz + kGhost)) return;   // may wrap through z = 0 / L
    lo = std::max(a, 0);
    hi = std::min(b, g.Z - 1);
}

// ---- the phases of one step; each returns the number of kernel launches ----
// part 0: the whole push; with z slabs part 1 = sort + the boundary supercell
// layers + the tail kernel + migration headers (everything the step's first
// exchange needs), part 2 = the interior layers (run while that exchange is
// in flight) + the check that none of them migrated
int phase_push(pic_ctx *ctx, bool sort_now, int jcur, bool profile, int part = 0)
{
    const Layout &L = ctx->L;
    const GridDev &g = L.g;
    int launches = 0;
    if (sort_now && part != 2) {
        StageMark m(ctx, 0, profile);
        for (int s = 0; s < ctx->cfg.n_species; ++s)
            if (ctx->has_particles[s]) {
                sort_particles(g, ctx->A[s], ctx->B[s], ctx->dev_n + s, L.cap[s], ctx->sort, ctx->sc_off[s],
                               ctx->err, ctx->st, &launches, ctx->occ_trim && part == 0 ? ctx->push_zr : nullptr);
                if (ctx->use_tile) {   // the fused kernel never touches ids
                    launch_copy_ids(ctx->B[s].id, ctx->A[s].id, ctx->dev_n + s, L.cap[s], ctx->st);
                    ++launches;
                }
            }
    }
    if (sort_now && part == 0 && ctx->occ_trim) enqueue_occ_range(ctx);
    StageMark m(ctx, 1, profile);
    // u^2 bounds: this step reads parity jcur (its J-tile scales were prepared by
    // the previous step's k_e_full or by ensure_prep), writes parity 1 - jcur
    if (ctx->use_tile) {
        // species go in pairs: one launch walks both species of a supercell in
        // one particle loop, so its E/B tile load, J-tile zeroing and flush,
        // its ragged last iteration and (C5) the CTAs of empty supercells are
        // paid once (C3 4.74 -> 4.43, C5_1g 4.38 -> 4.02 ms per step)
        TileSpecies ts{};
        int64_t cap_total = 0;
        for (int s = 0; s < ctx->cfg.n_species; ++s) {
            if (!ctx->has_particles[s]) continue;
            ts.in[ts.n] = sort_now ? ctx->B[s] : ctx->A[s];
            ts.pm[ts.n] = ctx->pmap[s][sort_now ? 1 : 0];
            ts.out[ts.n] = ctx->A[s];
            ts.sc_off[ts.n] = ctx->sc_off[s];
            ts.sp[ts.n] = species_dev(ctx, s, jcur);
            cap_total += L.cap[s];
            ++ts.n;
            if (ts.n == 2) {   // a launch takes one or two species
                launch_push_tile(ctx->eb_map, g, ctx->EB, ctx->J[jcur], ts, ctx->err,
                                 cap_total / std::max<int64_t>(1, L.n_sc), part, ctx->zb, ctx->push_zr, ctx->st);
                ++launches;
                if (profile) ctx->particle_launches++;
                ts.n = 0;
                cap_total = 0;
            }
        }
        if (ts.n > 0) {
            launch_push_tile(ctx->eb_map, g, ctx->EB, ctx->J[jcur], ts, ctx->err,
                             cap_total / std::max<int64_t>(1, L.n_sc), part, ctx->zb, ctx->push_zr, ctx->st);
            ++launches;
            if (profile) ctx->particle_launches++;
        }
    }
    for (int s = 0; s < ctx->cfg.n_species; ++s) {
        if (!ctx->has_particles[s]) continue;
        const SpeciesDev sp = species_dev(ctx, s, jcur);
        if (!ctx->use_tile && part != 2) {
            const ParticlesDev &in = sort_now ? ctx->B[s] : ctx->A[s];
            launch_push_tail(g, ctx->EB, ctx->J[jcur], in, ctx->A[s], nullptr, ctx->dev_n + s, L.cap[s], sp,
                             sort_now, ctx->err, ctx->st);
            ++launches;
            if (profile) ctx->particle_launches++;
        }
        if (ctx->slabs && part != 2) {
            if (ctx->use_tile) {   // particles received since the last sort (none right after it)
                if (!sort_now) {
                    launch_push_tail(g, ctx->EB, ctx->J[jcur], ctx->A[s], ctx->A[s], ctx->sc_off[s] + L.n_sc,
                                     ctx->dev_n + s, 4 * L.mig, sp, false, ctx->err, ctx->st);
                    ++launches;
                }
            }
            launch_mig_finalize(ctx->mig[s], ctx->err, ctx->st);
            ++launches;
        }
        if (ctx->slabs && part == 2 && ctx->use_tile) {
            launch_mig_late_check(ctx->mig[s], ctx->err, ctx->st);
            ++launches;
        }
    }
    return launches;
}

// Supercell layers per slab end whose particles may, this step, deposit into
// the exchanged J ghost planes or leave the slab: a particle moves less than
// c dt per step on each axis, so one sorted into layer l >= zb (z >= zb S dz
// above the slab's lower face) is still at z >= dz after the <= K - 1 steps
// since the sort, and its path of this step stays inside [0, nz) -- no
// deposit below plane 0, no migration; likewise at the upper face.  Without
// periodic re-sorts (K = 0) every layer is a boundary layer.
int boundary_layers(const pic_config &c, const GridDev &g)
{
    if (c.sort_every <= 0) return g.nsz;
    const double drift = (double)(c.sort_every - 1) * c.c * c.dt / c.dz;   // cells
    const int zb = (int)std::ceil((1.0 + drift) / g.S + 1e-12);
    return std::min(zb, g.nsz);
}

// J-tile scale preparation from the u^2 bound of parity `from` (the step that
// was pushed last), resetting the other parity for the next push
StepPrep make_prep(const pic_ctx *ctx, int from)
{
    StepPrep p{};
    p.n_species = (int)ctx->cfg.n_species;
    for (int s = 0; s < p.n_species; ++s) p.qw[s] = ctx->cfg.q[s] * ctx->cfg.w[s];
    p.c = ctx->L.g.c;
    p.dV = ctx->L.g.dx * ctx->L.g.dy * ctx->L.g.dz;
    p.u2max_in = ctx->u2max[from];
    p.u2max_out = ctx->u2max[1 - from];
    p.scale = ctx->tile_scale;
    return p;
}

// before the first step after new particles: the stand-alone preparation
void ensure_prep(pic_ctx *ctx)
{
    if (ctx->prep_ready) return;
    launch_step_prep(make_prep(ctx, ctx->jcur), ctx->st);
    ctx->launches += 1;
    ctx->prep_ready = true;
}

int phase_fields_e(pic_ctx *ctx, int jcur, bool profile)
{
    const GridDev &g = ctx->L.g;
    StageMark m(ctx, 2, profile);
    int launches = 0;
    if (ctx->slabs) {
        launch_j_ghost_add(g, ctx->J[jcur], ctx->jrecv[0], ctx->jrecv[1], ctx->st);
        ++launches;
        for (int s = 0; s < ctx->cfg.n_species; ++s) {
            launch_mig_append(ctx->mrecv[s][0], ctx->mrecv[s][1], (int)ctx->L.mig, ctx->A[s], ctx->dev_n + s,
                              ctx->L.cap[s], ctx->err, ctx->st);
            launches += 2;
        }
    }
    // B^{n+1/2} is already in Bh (written by the previous step's phase_fields_b)
    if (g.open_lo) {
        launch_laser_coeffs(g, ctx->laser_par, ctx->dev_step, ctx->laser, ctx->st);
        ++launches;
    }
    // + the next step's J-tile scales from this step's bound (parity 1 - jcur)
    JPlanes jl;
    j_planes(ctx, ctx->push_zr, jl.cur_lo, jl.cur_hi);
    j_planes(ctx, ctx->prev_zr, jl.next_lo, jl.next_hi);
    launch_e_full(g, ctx->EB, ctx->Bh, ctx->J[jcur], ctx->J[1 - jcur], make_prep(ctx, 1 - jcur), ctx->st, jl);
    return launches + 1;
}

// slabs compute the lower ghost plane of Bh locally, except below an open face
// (it lies outside the box and stays 0)
int bh_kbegin(const pic_ctx *ctx) { return ctx->slabs && !ctx->L.g.open_lo ? -1 : 0; }

// the second half step of this step and the first half step of the next one
// in one pass: B^{n+1} -> EB, B^{n+3/2} -> Bh
int phase_fields_b(pic_ctx *ctx, bool profile)
{
    StageMark m(ctx, 2, profile);
    launch_b_half(ctx->L.g, ctx->EB, ctx->Bh, ctx->EB + 3 * ctx->L.g.cs, ctx->Bh, ctx->st, bh_kbegin(ctx));
    return 1;
}

// Bh = B^n - (c dt/2) curl E^n from EB (once after EB was set from the host);
// needs valid E ghosts
void refresh_bh(pic_ctx *ctx)
{
    if (!ctx->bh_stale) return;
    launch_b_half(ctx->L.g, ctx->EB, ctx->EB + 3 * ctx->L.g.cs, ctx->Bh, nullptr, ctx->st, bh_kbegin(ctx));
    ctx->launches += 1;
    ctx->bh_stale = false;
}

// a whole step on one rank (NCCL exchanges or none); returns launches or < 0
int enqueue_step(pic_ctx *ctx, bool sort_now, int jcur, bool profile)
{
    int launches = 0;
    if (ctx->slabs) {
        // boundary layers first; their J ghost planes and the migrating
        // particles go out on st_x while the interior layers are pushed on st
        launches += phase_push(ctx, sort_now, jcur, profile, 1);
        if (cudaEventRecord(ctx->ev_fork, ctx->st) != cudaSuccess ||
            cudaStreamWaitEvent(ctx->st_x, ctx->ev_fork, 0) != cudaSuccess)
            return -1;
        {
            cudaEvent_t a = nullptr;
            if (profile) {
                a = take_event(ctx);
                cudaEventRecord(a, ctx->st_x);
            }
            if (exchange_nccl(ctx, msgs_current(ctx, jcur), ctx->st_x) != PIC_OK) return -1;
            if (profile) {
                cudaEvent_t b = take_event(ctx);
                cudaEventRecord(b, ctx->st_x);
                ctx->ev_marks.push_back({3, {a, b}});
            }
        }
        if (cudaEventRecord(ctx->ev_join, ctx->st_x) != cudaSuccess) return -1;
        launches += phase_push(ctx, sort_now, jcur, profile, 2);
        if (cudaStreamWaitEvent(ctx->st, ctx->ev_join, 0) != cudaSuccess) return -1;
    } else {
        launches += phase_push(ctx, sort_now, jcur, profile);
    }
    launches += phase_fields_e(ctx, jcur, profile);
    if (ctx->slabs) {
        StageMark m(ctx, 3, profile);
        if (exchange_nccl(ctx, msgs_fields(ctx, 0, 3)) != PIC_OK) return -1;
    }
    launches += phase_fields_b(ctx, profile);
    if (ctx->slabs) {
        StageMark m(ctx, 3, profile);
        if (exchange_nccl(ctx, msgs_fields(ctx, 3, 6)) != PIC_OK) return -1;
    }
    for (int s = 0; s < ctx->cfg.n_species; ++s) ctx->has_particles[s] = ctx->has_particles[s] || ctx->slabs;
    return launches;
}

void destroy_graphs(pic_ctx *ctx)
{
    for (auto &row : ctx->graph)
        for (auto &ge : row)
            if (ge) {
                cudaGraphExecDestroy(ge);
                ge = nullptr;
            }
    ctx->graphs_valid = false;
}

int build_graph(pic_ctx *ctx, bool sort_now, int jcur)
{
    cudaGraph_t graph;
    PIC_CUDA(ctx, cudaStreamBeginCapture(ctx->st, cudaStreamCaptureModeThreadLocal));
    const int n = enqueue_step(ctx, sort_now, jcur, false);
    cudaError_t e = cudaStreamEndCapture(ctx->st, &graph);
    if (n < 0) {
        if (e == cudaSuccess) cudaGraphDestroy(graph);
        return PIC_ENCCL;
    }
    if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaStreamEndCapture");
    e = cudaGraphInstantiate(&ctx->graph[sort_now][jcur], graph, 0);
    cudaGraphDestroy(graph);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaGraphInstantiate");
    ctx->graph_launches[sort_now][jcur] = n;
    ctx->graph_zr[sort_now][jcur][0] = ctx->push_zr[0];
    ctx->graph_zr[sort_now][jcur][1] = ctx->push_zr[1];
    ctx->graph_zr[sort_now][jcur][2] = ctx->prev_zr[0];
    ctx->graph_zr[sort_now][jcur][3] = ctx->prev_zr[1];
    return PIC_OK;
}

// TMA tensor map of the E/B fields: 4-D (x, y, z, component), box = one
// supercell tile with halo (x extent padded to the shared row pitch) x 6,
// no swizzle; box nodes past the padded array's x end are zero-filled and
// never used.
int encode_eb_map(pic_ctx *ctx)
{
    void *fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !fn)
        return fail(ctx, PIC_ECUDA, "cuTensorMapEncodeTiled unavailable");
    auto encode = (PFN_cuTensorMapEncodeTiled_v12000)fn;
    const GridDev &g = ctx->L.g;
    int bx[4];
    tile_box(g.S, g.H, bx);
    cuuint64_t dims[4] = {(cuuint64_t)g.X, (cuuint64_t)g.Y, (cuuint64_t)g.Z, 6};
    cuuint64_t strides[3] = {sizeof(double) * (cuuint64_t)g.X, sizeof(double) * (cuuint64_t)g.X * g.Y,
                             sizeof(double) * (cuuint64_t)g.cs};
    cuuint32_t box[4] = {(cuuint32_t)bx[0], (cuuint32_t)bx[1], (cuuint32_t)bx[2], (cuuint32_t)bx[3]};
    cuuint32_t estr[4] = {1, 1, 1, 1};
    CUresult r = encode(&ctx->eb_map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, ctx->EB, dims, strides, box,
                        estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(ctx, PIC_ECUDA, "cuTensorMapEncodeTiled failed");
    return PIC_OK;
}

// The particle stores as 2-D tensors [6 components][cap + 2 nodes] (the
// SoA columns x, y, z, ux, uy, uz at a constant pitch) with a box of
// [6][kPartBox]: the fused kernel stages a warp's particles with one load.
int encode_particle_maps(pic_ctx *ctx)
{
    void *fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !fn)
        return fail(ctx, PIC_ECUDA, "cuTensorMapEncodeTiled unavailable");
    auto encode = (PFN_cuTensorMapEncodeTiled_v12000)fn;
    for (int s = 0; s < ctx->cfg.n_species; ++s)
        for (int k = 0; k < 2; ++k) {
            const ParticlesDev &P = k ? ctx->B[s] : ctx->A[s];
            cuuint64_t dims[2] = {(cuuint64_t)ctx->L.cap[s] + 2, 6};
            cuuint64_t strides[1] = {(cuuint64_t)particle_col_bytes(ctx->L.cap[s])};
            cuuint32_t box[2] = {(cuuint32_t)kPartBox, 6};
            cuuint32_t estr[2] = {1, 1};
            CUresult r = encode(&ctx->pmap[s][k], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, P.x, dims, strides, box, estr,
                                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            if (r != CUDA_SUCCESS) return fail(ctx, PIC_ECUDA, "cuTensorMapEncodeTiled (particles) failed");
        }
    return PIC_OK;
}

int check_device_error(pic_ctx *ctx)
{
    unsigned h = 0;
    PIC_CUDA(ctx, cudaMemcpyAsync(&h, ctx->err, sizeof(unsigned), cudaMemcpyDeviceToHost, ctx->st));
    PIC_CUDA(ctx, cudaStreamSynchronize(ctx->st));
    if (h & kErrNonFinite) return fail(ctx, PIC_ENONFINITE, "non-finite particle state");
    if (h & kErrDisplacement) return fail(ctx, PIC_EDISPLACEMENT, "displacement >= 1 cell");
    if (h & kErrRange) return fail(ctx, PIC_EINVAL, "particle position outside the domain / slab");
    if (h & kErrCapacity) return fail(ctx, PIC_ECAPACITY, "device capacity exceeded (particles or migration)");
    if (h & kErrCheck) return fail(ctx, PIC_ECUDA, "internal index check failed (PIC_CHECK build)");
    if (h & kErrLateMigration)
        return fail(ctx, PIC_ECUDA, "an interior supercell layer's particle left the slab (overlap bound violated)");
    return PIC_OK;
}

void collect_profile(pic_ctx *ctx)
{
    for (auto &m : ctx->ev_marks) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, m.second.first, m.second.second);
        ctx->stage_ms[m.first] += ms;
    }
    ctx->ev_marks.clear();
    ctx->ev_used = 0;
}

// ---- diagnostics (diag.cu); between steps, so jrecv is free scratch ----
double *diag_rho_below(pic_ctx *ctx) { return ctx->jrecv[0]; }
double *diag_jz_below(pic_ctx *ctx) { return ctx->jrecv[0] + plane_pair(ctx->L.g); }

// the top ghost node pair of rho (charge of nodes owned by the slab above)
// and the top interior Jz pair go up
std::vector<Msg> msgs_diag(pic_ctx *ctx)
{
    const GridDev &g = ctx->L.g;
    const double *Jz = ctx->J[ctx->jlast] + 2 * g.cs;
    return {{ctx->rho + plane_off(g, g.nz), diag_rho_below(ctx), plane_pair(g), 1},
            {(double *)Jz + plane_off(g, g.nz - 2), diag_jz_below(ctx), plane_pair(g), 1}};
}

int diag_particles(pic_ctx *ctx)
{
    const GridDev &g = ctx->L.g;
    PIC_CUDA(ctx, cudaMemsetAsync(ctx->rho, 0, sizeof(double) * (size_t)g.cs, ctx->st));
    PIC_CUDA(ctx, cudaMemsetAsync(ctx->acc, 0, sizeof(double) * kAccSlots, ctx->st));
    for (int s = 0; s < ctx->cfg.n_species; ++s) {
        launch_diag_particles(g, ctx->A[s], ctx->dev_n + s, ctx->L.cap[s], ctx->cfg.q[s] * ctx->cfg.w[s],
                              ctx->rho, ctx->acc + 9 + s, ctx->st);
        ctx->launches += 2;
    }
    PIC_CUDA(ctx, cudaGetLastError());
    return PIC_OK;
}

int diag_nodes(pic_ctx *ctx, pic_diag *out, double *rho_host)
{
    const GridDev &g = ctx->L.g;
    const bool have_prev = ctx->diag_last_step == ctx->step_index - 1;
    launch_diag_nodes(g, ctx->EB, ctx->J[ctx->jlast], ctx->slabs ? diag_jz_below(ctx) + (size_t)g.X * g.Y : nullptr,
                      ctx->rho, ctx->slabs ? diag_rho_below(ctx) : nullptr, ctx->rho_prev, ctx->gauss0,
                      have_prev, ctx->diag_have_g0, ctx->acc, ctx->st);
    ctx->launches += 2;
    PIC_CUDA(ctx, cudaGetLastError());
    double a[kAccSlots];
    PIC_CUDA(ctx, cudaMemcpyAsync(a, ctx->acc, sizeof(a), cudaMemcpyDeviceToHost, ctx->st));
    if (rho_host) {
        cudaMemcpy3DParms p = {};
        p.srcPtr = make_cudaPitchedPtr((void *)ctx->rho, sizeof(double) * g.X, g.X, g.Y);
        p.srcPos = make_cudaPos(sizeof(double) * kGhost, kGhost, kGhost);
        p.dstPtr = make_cudaPitchedPtr(rho_host, sizeof(double) * g.nx, g.nx, g.ny);
        p.extent = make_cudaExtent(sizeof(double) * g.nx, g.ny, g.nz);
        p.kind = cudaMemcpyDeviceToHost;
        PIC_CUDA(ctx, cudaMemcpy3DAsync(&p, ctx->st));
    }
    PIC_CUDA(ctx, cudaStreamSynchronize(ctx->st));
    const double dV = g.dx * g.dy * g.dz;
    pic_diag d{};
    d.step = ctx->step_index;
    d.field_energy = a[0] * dV / (8.0 * M_PI);
    for (int s = 0; s < PIC_MAX_SPECIES; ++s)
        d.kinetic_energy[s] = s < ctx->cfg.n_species ? a[9 + s] * ctx->cfg.w[s] * ctx->cfg.m[s] * g.c * g.c : 0.0;
    d.charge = a[1] * dV;
    for (int c = 0; c < 3; ++c) d.current[c] = a[2 + c] * dV;
    d.max_div_b = a[5];
    d.max_gauss = a[6];
    d.max_gauss_drift = ctx->diag_have_g0 ? a[7] : 0.0;
    d.max_continuity = have_prev ? a[8] : -1.0;
    ctx->diag_have_g0 = true;
    ctx->diag_last_step = ctx->step_index;
    if (out) *out = d;
    return PIC_OK;
}

}  // namespace

extern "C" {

int pic_workspace_size(const pic_config *cfg, size_t *bytes)
{
    const std::string v = validate(cfg);
    if (!v.empty() || !bytes) return PIC_EINVAL;
    *bytes = make_layout(cfg).total;
    return PIC_OK;
}

int pic_nccl_unique_id(uint8_t id[128])
{
    if (!id) return PIC_EINVAL;
    NcclApi *api = nccl_api();
    if (!api) return PIC_ENCCL;
    ncclUniqueId u;
    if (api->getUniqueId(&u) != ncclSuccess) return PIC_ENCCL;
    static_assert(sizeof(u) == 128, "ncclUniqueId size");
    memcpy(id, &u, 128);
    return PIC_OK;
}

int pic_init(const pic_config *cfg, void *d_workspace, size_t bytes, pic_ctx **out)
{
    if (!out) return PIC_EINVAL;
    *out = nullptr;
    const std::string v = validate(cfg);
    if (!v.empty()) return PIC_EINVAL;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return PIC_ECUDA;
    Layout L = make_layout(cfg);
    if (!d_workspace || bytes < L.total) return PIC_ENOMEM;
    if (((uintptr_t)d_workspace) % kAlign) return PIC_EINVAL;
    pic_ctx *ctx = new pic_ctx();
    ctx->cfg = *cfg;
    ctx->L = L;
    ctx->ws = (char *)d_workspace;
    ctx->st = (cudaStream_t)cfg->stream;
    ctx->slabs = cfg->nranks > 1;
    ctx->local_group = ctx->slabs && (cfg->flags & PIC_FLAG_LOCAL_GROUP);
    ctx->EB = (double *)(ctx->ws + L.off_eb);
    ctx->Bh = (double *)(ctx->ws + L.off_bh);
    ctx->J[0] = (double *)(ctx->ws + L.off_j[0]);
    ctx->J[1] = (double *)(ctx->ws + L.off_j[1]);
    ctx->u2max[0] = (unsigned *)(ctx->ws + L.off_stat);
    ctx->u2max[1] = ctx->u2max[0] + PIC_MAX_SPECIES;
    ctx->dev_n = (int64_t *)(ctx->ws + L.off_n);
    unsigned *mcnt = (unsigned *)(ctx->ws + L.off_mcnt);
    for (int s = 0; s < cfg->n_species; ++s) {
        ctx->A[s] = carve_particles(ctx->ws, L.off_sp[s][0], L.cap[s]);
        ctx->B[s] = carve_particles(ctx->ws, L.off_sp[s][1], L.cap[s]);
        ctx->sc_off[s] = (int64_t *)(ctx->ws + L.off_scoff[s]);
        ctx->mig[s].cap = (int)L.mig;
        ctx->mig[s].count = mcnt + 2 * s;
        for (int d = 0; d < 2; ++d) {
            ctx->mig[s].send[d] = L.mig ? (double *)(ctx->ws + L.off_msend[s][d]) : nullptr;
            ctx->mrecv[s][d] = L.mig ? (double *)(ctx->ws + L.off_mrecv[s][d]) : nullptr;
        }
    }
    for (int d = 0; d < 2; ++d) ctx->jrecv[d] = L.mig ? (double *)(ctx->ws + L.off_jrecv[d]) : nullptr;
    ctx->sort.key = (uint32_t *)(ctx->ws + L.off_key);
    ctx->sort.slot = (uint32_t *)(ctx->ws + L.off_slot);
    ctx->sort.perm_tmp = (uint32_t *)(ctx->ws + L.off_perm_tmp);
    ctx->sort.perm = (uint32_t *)(ctx->ws + L.off_perm);
    ctx->sort.count = (uint32_t *)(ctx->ws + L.off_count);
    ctx->sort.start = (uint32_t *)(ctx->ws + L.off_start);
    ctx->sort.block_sums = (uint32_t *)(ctx->ws + L.off_bsums);
    ctx->err = (unsigned *)(ctx->ws + L.off_err);
    ctx->rho = (double *)(ctx->ws + L.off_rho);
    ctx->rho_prev = (double *)(ctx->ws + L.off_rho_prev);
    ctx->gauss0 = (double *)(ctx->ws + L.off_gauss0);
    ctx->acc = (double *)(ctx->ws + L.off_acc);
    ctx->laser = (double *)(ctx->ws + L.off_laser);
    ctx->dev_step = (int64_t *)(ctx->ws + L.off_step);
    ctx->tile_scale = (double *)(ctx->ws + L.off_scale);
    ctx->L.g.laser = ctx->laser;
    ctx->laser_par[0] = cfg->laser_e0;
    ctx->laser_par[1] = cfg->laser_omega;
    ctx->laser_par[2] = cfg->laser_ramp;
    ctx->laser_par[3] = cfg->laser_t0;
    ctx->laser_par[4] = cfg->laser_pol[0];
    ctx->laser_par[5] = cfg->laser_pol[1];
    ctx->use_tile = !(cfg->flags & PIC_FLAG_NAIVE) && tile_supported((int)cfg->supercell, ctx->L.g.H);
    configure_tile_kernels();
    {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, dev);
    }
    if (ctx->use_tile && (encode_eb_map(ctx) != PIC_OK || encode_particle_maps(ctx) != PIC_OK)) {
        delete ctx;
        return PIC_ECUDA;
    }
    // zero fields, offsets, counters and the error word (particle arrays stay
    // garbage until set; the exchange buffers are written before being read)
    cudaError_t e = cudaMemsetAsync(ctx->ws, 0, L.off_sp[0][0], ctx->st);
    for (int s = 0; e == cudaSuccess && s < cfg->n_species; ++s)
        e = cudaMemsetAsync(ctx->sc_off[s], 0, sizeof(int64_t) * (size_t)(L.n_sc + 1), ctx->st);
    if (e == cudaSuccess) e = cudaMemsetAsync(ctx->ws + L.off_err, 0, L.total - L.off_err, ctx->st);
    // receive buffers: a face of an open box never receives, so they must read 0
    for (int s = 0; e == cudaSuccess && s < cfg->n_species; ++s)
        for (int d = 0; e == cudaSuccess && d < 2; ++d)
            if (ctx->mrecv[s][d]) e = cudaMemsetAsync(ctx->mrecv[s][d], 0, sizeof(double) * (1 + 7 * (size_t)L.mig), ctx->st);
    for (int d = 0; e == cudaSuccess && d < 2; ++d)
        if (ctx->jrecv[d]) e = cudaMemsetAsync(ctx->jrecv[d], 0, sizeof(double) * 3 * 2 * (size_t)L.g.X * L.g.Y, ctx->st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->st);
    if (e != cudaSuccess) {
        delete ctx;
        return PIC_ECUDA;
    }
    ctx->push_zr[1] = L.g.nsz;   // every layer unless trimmed (push_layers)
    ctx->occ_trim = ctx->use_tile && !ctx->slabs;
    if (ctx->occ_trim && (cudaHostAlloc((void **)&ctx->h_occ, 2 * sizeof(int), cudaHostAllocMapped) != cudaSuccess ||
                          cudaHostGetDevicePointer((void **)&ctx->d_occ, ctx->h_occ, 0) != cudaSuccess ||
                          cudaEventCreateWithFlags(&ctx->ev_occ, cudaEventDisableTiming) != cudaSuccess)) {
        pic_destroy(ctx);
        return PIC_ECUDA;
    }
    if (ctx->slabs) {
        ctx->zb = boundary_layers(*cfg, L.g);
        if (!ctx->local_group &&
            (cudaStreamCreateWithFlags(&ctx->st_x, cudaStreamNonBlocking) != cudaSuccess ||
             cudaEventCreateWithFlags(&ctx->ev_fork, cudaEventDisableTiming) != cudaSuccess ||
             cudaEventCreateWithFlags(&ctx->ev_join, cudaEventDisableTiming) != cudaSuccess)) {
            pic_destroy(ctx);
            return PIC_ECUDA;
        }
    }
    if (ctx->slabs && !ctx->local_group) {
        NcclApi *api = nccl_api();
        ncclUniqueId id;
        memcpy(&id, cfg->nccl_id, 128);
        if (!api || api->commInitRank(&ctx->comm, (int)cfg->nranks, id, (int)cfg->rank) != ncclSuccess) {
            pic_destroy(ctx);
            return PIC_ENCCL;
        }
    }
    *out = ctx;
    return PIC_OK;
}

int pic_set_particles(pic_ctx *ctx, int species, int64_t n, const double *x, const double *y,
                      const double *z, const double *ux, const double *uy, const double *uz,
                      const uint64_t *id)
{
    if (!ctx) return PIC_EINVAL;
    if (species < 0 || species >= ctx->cfg.n_species) return fail(ctx, PIC_EINVAL, "bad species");
    if (n < 0 || (n > 0 && !(x && y && z && ux && uy && uz && id)))
        return fail(ctx, PIC_EINVAL, "bad particle arrays");
    const GridDev &g = ctx->L.g;
    const char *outside = g.open_z ? "particle position outside [0, Lx) x [0, Ly) x [0, (nz-1) dz)"
                                   : "particle position outside [0, L)";
    // slabs select their particles on the host, so they check there; a single
    // domain leaves the check to the device (the sort's key pass flags any
    // position outside the box), which keeps the host out of the upload path
    if (ctx->slabs)
        for (int64_t p = 0; p < n; ++p)
            if (!(x[p] >= 0.0 && x[p] < g.Lx && y[p] >= 0.0 && y[p] < g.Ly && z[p] >= 0.0 && z[p] < g.zmax))
                return fail(ctx, PIC_EINVAL, outside);
    const double *src[6] = {x, y, z, ux, uy, uz};
    std::vector<double> sel[6];
    std::vector<uint64_t> sel_id;
    int64_t m = n;
    if (ctx->slabs) {   // keep the particles of this rank's slab
        for (int c = 0; c < 6; ++c) sel[c].reserve((size_t)(n / ctx->cfg.nranks + 16));
        for (int64_t p = 0; p < n; ++p)
            if (z[p] >= g.zlo && z[p] < g.zhi) {
                for (int c = 0; c < 6; ++c) sel[c].push_back(src[c][p]);
                sel_id.push_back(id[p]);
            }
        m = (int64_t)sel_id.size();
        for (int c = 0; c < 6; ++c) src[c] = sel[c].data();
        id = sel_id.data();
    }
    if (m > ctx->L.cap[species]) return fail(ctx, PIC_ECAPACITY, "n exceeds capacity");
    if (!ctx->slabs) PIC_CUDA(ctx, cudaMemsetAsync(ctx->err, 0, sizeof(unsigned), ctx->st));   // fresh check
    const ParticlesDev &Bs = ctx->B[species];
    double *dst[6] = {Bs.x, Bs.y, Bs.z, Bs.ux, Bs.uy, Bs.uz};
    for (int c = 0; c < 6 && m > 0; ++c)
        PIC_CUDA(ctx, cudaMemcpyAsync(dst[c], src[c], sizeof(double) * (size_t)m, cudaMemcpyHostToDevice, ctx->st));
    if (m > 0)
        PIC_CUDA(ctx, cudaMemcpyAsync(Bs.id, id, sizeof(uint64_t) * (size_t)m, cudaMemcpyHostToDevice, ctx->st));
    PIC_CUDA(ctx, cudaMemcpyAsync(ctx->dev_n + species, &m, sizeof(int64_t), cudaMemcpyHostToDevice, ctx->st));
    ctx->has_particles[species] = m > 0 || ctx->slabs;
    int launches = 0;
    sort_particles(g, Bs, ctx->A[species], ctx->dev_n + species, std::max<int64_t>(m, 1), ctx->sort,
                   ctx->sc_off[species], ctx->err, ctx->st, &launches);
    launch_u2max(ctx->A[species], m, ctx->u2max[ctx->jcur] + species, ctx->st);
    ctx->prep_ready = false;
    ctx->launches += launches + 1;
    if (!ctx->slabs) {   // the device-side range check of the key pass
        unsigned h = 0;
        PIC_CUDA(ctx, cudaMemcpyAsync(&h, ctx->err, sizeof(unsigned), cudaMemcpyDeviceToHost, ctx->st));
        PIC_CUDA(ctx, cudaStreamSynchronize(ctx->st));
        if (h & (kErrRange | kErrNonFinite)) {   // reject: the species is left empty
            const int64_t zero = 0;
            PIC_CUDA(ctx, cudaMemsetAsync(ctx->err, 0, sizeof(unsigned), ctx->st));
            PIC_CUDA(ctx, cudaMemcpyAsync(ctx->dev_n + species, &zero, sizeof(int64_t), cudaMemcpyHostToDevice,
                                          ctx->st));
            PIC_CUDA(ctx, cudaMemsetAsync(ctx->sc_off[species], 0, sizeof(int64_t) * (size_t)(ctx->L.n_sc + 1),
                                          ctx->st));
            PIC_CUDA(ctx, cudaStreamSynchronize(ctx->st));
            ctx->has_particles[species] = false;
            destroy_graphs(ctx);
            return fail(ctx, PIC_EINVAL, outside);
        }
    }
    if (ctx->occ_trim) {
        enqueue_occ_range(ctx);
        PIC_CUDA(ctx, cudaEventRecord(ctx->ev_occ, ctx->st));
        ctx->occ_pending = true;
        int rc = poll_occ(ctx, true);
        if (rc != PIC_OK) return rc;
    }
    PIC_CUDA(ctx, cudaGetLastError());
    destroy_graphs(ctx);
    return check_device_error(ctx);
}

int pic_set_fields6(pic_ctx *ctx, const double *const f[6])
{
    if (!ctx || !f) return PIC_EINVAL;
    for (int c = 0; c < 6; ++c)
        if (!f[c]) return fail(ctx, PIC_EINVAL, "pic_set_fields6: NULL component");
    const GridDev &g = ctx->L.g;
    for (int c = 0; c < 6; ++c) {
        cudaMemcpy3DParms p = {};
        p.srcPtr = make_cudaPitchedPtr((void *)f[c], sizeof(double) * g.nx, g.nx, g.ny);
        p.dstPtr = make_cudaPitchedPtr(ctx->EB + c * g.cs, sizeof(double) * g.X, g.X, g.Y);
        p.dstPos = make_cudaPos(sizeof(double) * kGhost, kGhost, kGhost);
        p.extent = make_cudaExtent(sizeof(double) * g.nx, g.ny, g.nz);
        p.kind = cudaMemcpyHostToDevice;
        PIC_CUDA(ctx, cudaMemcpy3DAsync(&p, ctx->st));
    }
    launch_fill_ghosts(g, ctx->EB, 6, ctx->st);
    ctx->launches += 1;
    ctx->ghosts_stale = ctx->slabs;   // z ghost planes come from the neighbours
    ctx->bh_stale = true;
    PIC_CUDA(ctx, cudaGetLastError());
    PIC_CUDA(ctx, cudaStreamSynchronize(ctx->st));
    return PIC_OK;
}

int pic_set_fields(pic_ctx *ctx, const double *f)
{
    if (!ctx || !f) return PIC_EINVAL;
    const GridDev &g = ctx->L.g;
    const size_t n = (size_t)g.nx * g.ny * g.nz;
    const double *const comp[6] = {f, f + n, f + 2 * n, f + 3 * n, f + 4 * n, f + 5 * n};
    return pic_set_fields6(ctx, comp);
}

int pic_get_fields9(pic_ctx *ctx, double *const f[9])
{
    if (!ctx || !f) return PIC_EINVAL;
    const GridDev &g = ctx->L.g;
    for (int c = 0; c < 9; ++c) {
        if (!f[c]) continue;
        const double *srcbase = c < 6 ? ctx->EB + c * g.cs : ctx->J[ctx->jlast] + (c - 6) * g.cs;
        cudaMemcpy3DParms p = {};
        p.srcPtr = make_cudaPitchedPtr((void *)srcbase, sizeof(double) * g.X, g.X, g.Y);
        p.srcPos = make_cudaPos(sizeof(double) * kGhost, kGhost, kGhost);
        p.dstPtr = make_cudaPitchedPtr(f[c], sizeof(double) * g.nx, g.nx, g.ny);
        p.extent = make_cudaExtent(sizeof(double) * g.nx, g.ny, g.nz);
        p.kind = cudaMemcpyDeviceToHost;
        PIC_CUDA(ctx, cudaMemcpy3DAsync(&p, ctx->st));
    }
    PIC_CUDA(ctx, cudaStreamSynchronize(ctx->st));
    return PIC_OK;
}

int pic_get_fields(pic_ctx *ctx, double *f)
{
    if (!ctx || !f) return PIC_EINVAL;
    const GridDev &g = ctx->L.g;
    const size_t n = (size_t)g.nx * g.ny * g.nz;
    double *const comp[9] = {f, f + n, f + 2 * n, f + 3 * n, f + 4 * n, f + 5 * n, f + 6 * n, f + 7 * n, f + 8 * n};
    return pic_get_fields9(ctx, comp);
}

static int device_slots(pic_ctx *ctx, int species, int64_t *n)
{
    PIC_CUDA(ctx, cudaMemcpyAsync(n, ctx->dev_n + species, sizeof(int64_t), cudaMemcpyDeviceToHost, ctx->st));
    PIC_CUDA(ctx, cudaStreamSynchronize(ctx->st));
    return PIC_OK;
}

int pic_get_particles(pic_ctx *ctx, int species, int64_t *n_inout, double *x, double *y, double *z,
                      double *ux, double *uy, double *uz, uint64_t *id)
{
    if (!ctx || !n_inout) return PIC_EINVAL;
    if (species < 0 || species >= ctx->cfg.n_species) return fail(ctx, PIC_EINVAL, "bad species");
    int64_t slots = 0;
    int rc = device_slots(ctx, species, &slots);
    if (rc != PIC_OK) return rc;
    const ParticlesDev &A = ctx->A[species];
    const double *src[6] = {A.x, A.y, A.z, A.ux, A.uy, A.uz};
    double *dst[6] = {x, y, z, ux, uy, uz};
    const int64_t capacity = *n_inout;
    if (!ctx->slabs && !ctx->L.g.open_z) {   // every slot is live
        *n_inout = slots;
        if (capacity < slots) return fail(ctx, PIC_ECAPACITY, "output arrays too small");
        for (int c = 0; c < 6 && slots > 0; ++c)
            if (dst[c])
                PIC_CUDA(ctx, cudaMemcpyAsync(dst[c], src[c], sizeof(double) * (size_t)slots,
                                              cudaMemcpyDeviceToHost, ctx->st));
        if (id && slots > 0)
            PIC_CUDA(ctx, cudaMemcpyAsync(id, A.id, sizeof(uint64_t) * (size_t)slots, cudaMemcpyDeviceToHost, ctx->st));
        PIC_CUDA(ctx, cudaStreamSynchronize(ctx->st));
        return PIC_OK;
    }
    // slabs / open z: skip the dead slots (x == -1) left by migration or
    // absorption -- a stable device compaction into B (free between steps)
    const ParticlesDev &Bs = ctx->B[species];
    const int64_t live = compact_live(A, Bs, slots, ctx->sort, (uint32_t *)(ctx->ws + ctx->L.off_bsums2), ctx->st);
    ctx->launches += 5;
    PIC_CUDA(ctx, cudaGetLastError());
    *n_inout = live;
    if (capacity < live) return fail(ctx, PIC_ECAPACITY, "output arrays too small");
    const double *bsrc[6] = {Bs.x, Bs.y, Bs.z, Bs.ux, Bs.uy, Bs.uz};
    for (int c = 0; c < 6 && live > 0; ++c)
        if (dst[c])
            PIC_CUDA(ctx, cudaMemcpyAsync(dst[c], bsrc[c], sizeof(double) * (size_t)live, cudaMemcpyDeviceToHost,
                                          ctx->st));
    if (id && live > 0)
        PIC_CUDA(ctx, cudaMemcpyAsync(id, Bs.id, sizeof(uint64_t) * (size_t)live, cudaMemcpyDeviceToHost, ctx->st));
    PIC_CUDA(ctx, cudaStreamSynchronize(ctx->st));
    return PIC_OK;
}

int pic_get_count(pic_ctx *ctx, int species, int64_t *n)
{
    if (!ctx || !n || species < 0 || species >= ctx->cfg.n_species) return PIC_EINVAL;
    if (!ctx->slabs && !ctx->L.g.open_z) return device_slots(ctx, species, n);
    int64_t cap = 0;
    int rc = pic_get_particles(ctx, species, &cap, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr);
    if (rc != PIC_OK && rc != PIC_ECAPACITY) return rc;
    *n = cap;
    return PIC_OK;
}

int pic_get_step_index(pic_ctx *ctx, int64_t *n)
{
    if (!ctx || !n) return PIC_EINVAL;
    *n = ctx->step_index;
    return PIC_OK;
}

int pic_step(pic_ctx *ctx, int64_t nsteps)
{
    if (!ctx || nsteps < 0) return PIC_EINVAL;
    if (ctx->local_group) return fail(ctx, PIC_ESTATE, "PIC_FLAG_LOCAL_GROUP contexts step via pic_step_group");
    const int64_t K = ctx->cfg.sort_every;
    const bool profile = (ctx->cfg.flags & PIC_FLAG_PROFILE) != 0;
    const bool use_graph = !profile && !(ctx->cfg.flags & PIC_FLAG_NO_GRAPH) && ctx->st != nullptr;
    if (ctx->ghosts_stale && nsteps > 0) {
        std::vector<Msg> m = msgs_fields(ctx, 0, 6);
        int rc = exchange_nccl(ctx, m);
        if (rc != PIC_OK) return rc;
        ctx->ghosts_stale = false;
    }
    if (nsteps > 0) {
        refresh_bh(ctx);
        ensure_prep(ctx);
    }
    for (int64_t s = 0; s < nsteps; ++s) {
        const bool sort_now = K > 0 && (ctx->step_index % K) == 0;
        const int jc = ctx->jcur;
        if (ctx->occ_trim) {
            int rc = poll_occ(ctx, false);
            if (rc != PIC_OK) return rc;
        }
        push_layers(ctx, sort_now, ctx->push_zr);
        if (use_graph) {
            if (!ctx->graphs_valid) {
                destroy_graphs(ctx);
                ctx->graphs_valid = true;
            }
            cudaGraphExec_t &ge = ctx->graph[sort_now][jc];
            const int *gz = ctx->graph_zr[sort_now][jc];
            if (ge && (gz[0] != ctx->push_zr[0] || gz[1] != ctx->push_zr[1] || gz[2] != ctx->prev_zr[0] ||
                       gz[3] != ctx->prev_zr[1])) {   // the occupied layers changed
                cudaGraphExecDestroy(ge);
                ge = nullptr;
            }
            if (!ge) {
                int rc = build_graph(ctx, sort_now, jc);
                if (rc != PIC_OK) return rc;
            }
            PIC_CUDA(ctx, cudaGraphLaunch(ge, ctx->st));
            ctx->launches += ctx->graph_launches[sort_now][jc];
        } else {
            const int n = enqueue_step(ctx, sort_now, jc, profile);
            if (n < 0) return PIC_ENCCL;
            ctx->launches += n;
            PIC_CUDA(ctx, cudaGetLastError());
        }
        ctx->prev_zr[0] = ctx->push_zr[0];
        ctx->prev_zr[1] = ctx->push_zr[1];
        if (sort_now && ctx->occ_trim) {   // the sort's occupied range is on its way to h_occ
            PIC_CUDA(ctx, cudaEventRecord(ctx->ev_occ, ctx->st));
            ctx->occ_pending = true;
        }
        ctx->jlast = jc;
        ctx->jcur = 1 - jc;
        ctx->step_index++;
    }
    int rc = check_device_error(ctx);
    if (profile) collect_profile(ctx);
    return rc;
}

int pic_step_group(pic_ctx *const *ctxs, int n, int64_t nsteps)
{
    if (!ctxs || n < 1 || nsteps < 0) return PIC_EINVAL;
    for (int r = 0; r < n; ++r) {
        if (!ctxs[r] || !ctxs[r]->local_group || ctxs[r]->cfg.nranks != n || ctxs[r]->cfg.rank != r)
            return fail(ctxs[r], PIC_EINVAL, "pic_step_group needs PIC_FLAG_LOCAL_GROUP ranks 0..n-1");
    }
    auto all = [&](auto f) {
        std::vector<std::vector<Msg>> m(n);
        for (int r = 0; r < n; ++r) m[r] = f(ctxs[r]);
        return m;
    };
    if (ctxs[0]->ghosts_stale && nsteps > 0) {
        int rc = exchange_local(ctxs, n, all([](pic_ctx *c) { return msgs_fields(c, 0, 6); }));
        if (rc != PIC_OK) return rc;
        for (int r = 0; r < n; ++r) ctxs[r]->ghosts_stale = false;
    }
    if (nsteps > 0)
        for (int r = 0; r < n; ++r) {
            refresh_bh(ctxs[r]);
            ensure_prep(ctxs[r]);
        }
    for (int64_t s = 0; s < nsteps; ++s) {
        const int64_t K = ctxs[0]->cfg.sort_every;
        const bool sort_now = K > 0 && (ctxs[0]->step_index % K) == 0;
        const int jc = ctxs[0]->jcur;
        // the same boundary / exchange / interior order as a NCCL step (the
        // copies here are ordered on each context's stream)
        for (int r = 0; r < n; ++r) ctxs[r]->launches += phase_push(ctxs[r], sort_now, jc, false, 1);
        int rc = exchange_local(ctxs, n, all([jc](pic_ctx *c) { return msgs_current(c, jc); }));
        if (rc != PIC_OK) return rc;
        for (int r = 0; r < n; ++r) ctxs[r]->launches += phase_push(ctxs[r], sort_now, jc, false, 2);
        for (int r = 0; r < n; ++r) ctxs[r]->launches += phase_fields_e(ctxs[r], jc, false);
        rc = exchange_local(ctxs, n, all([](pic_ctx *c) { return msgs_fields(c, 0, 3); }));
        if (rc != PIC_OK) return rc;
        for (int r = 0; r < n; ++r) ctxs[r]->launches += phase_fields_b(ctxs[r], false);
        rc = exchange_local(ctxs, n, all([](pic_ctx *c) { return msgs_fields(c, 3, 6); }));
        if (rc != PIC_OK) return rc;
        for (int r = 0; r < n; ++r) {
            pic_ctx *c = ctxs[r];
            for (int sp = 0; sp < c->cfg.n_species; ++sp) c->has_particles[sp] = true;
            c->jlast = jc;
            c->jcur = 1 - jc;
            c->step_index++;
        }
    }
    int rc = PIC_OK;
    for (int r = 0; r < n; ++r) {
        PIC_CUDA(ctxs[r], cudaGetLastError());
        const int e = check_device_error(ctxs[r]);
        if (e != PIC_OK && rc == PIC_OK) rc = e;
    }
    return rc;
}

int pic_diagnostics(pic_ctx *ctx, pic_diag *out, double *rho)
{
    if (!ctx) return PIC_EINVAL;
    if (ctx->local_group) return fail(ctx, PIC_ESTATE, "PIC_FLAG_LOCAL_GROUP contexts use pic_diagnostics_group");
    if (ctx->L.g.open_z) return fail(ctx, PIC_EINVAL, "diagnostics assume a periodic z box");
    if (ctx->ghosts_stale) {
        int rc = exchange_nccl(ctx, msgs_fields(ctx, 0, 6));
        if (rc != PIC_OK) return rc;
        ctx->ghosts_stale = false;
    }
    int rc = diag_particles(ctx);
    if (rc == PIC_OK && ctx->slabs) rc = exchange_nccl(ctx, msgs_diag(ctx));
    if (rc == PIC_OK) rc = diag_nodes(ctx, out, rho);
    return rc;
}

int pic_diagnostics_group(pic_ctx *const *ctxs, int n, pic_diag *out, double *const *rho)
{
    if (!ctxs || n < 1) return PIC_EINVAL;
    for (int r = 0; r < n; ++r) {
        if (!ctxs[r] || !ctxs[r]->local_group || ctxs[r]->cfg.nranks != n || ctxs[r]->cfg.rank != r)
            return fail(ctxs[r], PIC_EINVAL, "pic_diagnostics_group needs PIC_FLAG_LOCAL_GROUP ranks 0..n-1");
    }
    if (ctxs[0]->L.g.open_z) return fail(ctxs[0], PIC_EINVAL, "diagnostics assume a periodic z box");
    auto all = [&](auto f) {
        std::vector<std::vector<Msg>> m(n);
        for (int r = 0; r < n; ++r) m[r] = f(ctxs[r]);
        return m;
    };
    if (ctxs[0]->ghosts_stale) {
        int rc = exchange_local(ctxs, n, all([](pic_ctx *c) { return msgs_fields(c, 0, 6); }));
        if (rc != PIC_OK) return rc;
        for (int r = 0; r < n; ++r) ctxs[r]->ghosts_stale = false;
    }
    for (int r = 0; r < n; ++r) {
        int rc = diag_particles(ctxs[r]);
        if (rc != PIC_OK) return rc;
    }
    int rc = exchange_local(ctxs, n, all([](pic_ctx *c) { return msgs_diag(c); }));
    if (rc != PIC_OK) return rc;
    for (int r = 0; r < n; ++r) {
        rc = diag_nodes(ctxs[r], out ? out + r : nullptr, rho ? rho[r] : nullptr);
        if (rc != PIC_OK) return rc;
    }
    return PIC_OK;
}

int pic_laser_preload(pic_ctx *ctx)
{
    if (!ctx) return PIC_EINVAL;
    if (!ctx->L.g.open_z) return fail(ctx, PIC_EINVAL, "pic_laser_preload needs bc_z == PIC_BC_OPEN");
    if (ctx->step_index != 0) return fail(ctx, PIC_ESTATE, "pic_laser_preload before the first step");
    launch_laser_preload(ctx->L.g, ctx->laser_par, ctx->EB, ctx->st);
    ctx->launches += 1;
    ctx->ghosts_stale = ctx->slabs;   // z ghost planes come from the neighbours
    ctx->bh_stale = true;
    PIC_CUDA(ctx, cudaGetLastError());
    PIC_CUDA(ctx, cudaStreamSynchronize(ctx->st));
    return PIC_OK;
}

int pic_balance_slabs(int64_t nz, int64_t nranks, int64_t granule, int64_t min_planes,
                      const double *plane_cost, int64_t *z_split)
{
    if (nz < 1 || nranks < 1 || granule < 1 || min_planes < 1 || !plane_cost || !z_split) return PIC_EINVAL;
    if (nz % granule) return PIC_EINVAL;
    const int64_t ng = nz / granule;                           // granules
    const int64_t mg = (min_planes + granule - 1) / granule;   // min granules per slab
    if (ng < nranks * mg) return PIC_EINVAL;
    std::vector<double> pre((size_t)ng + 1, 0.0);              // prefix cost over granules
    for (int64_t q = 0; q < ng; ++q) {
        double c = 0.0;
        for (int64_t k = q * granule; k < (q + 1) * granule; ++k) {
            if (!(plane_cost[k] >= 0.0) || !std::isfinite(plane_cost[k])) return PIC_EINVAL;
            c += plane_cost[k];
        }
        pre[(size_t)q + 1] = pre[(size_t)q] + c;
    }
    // Is a largest slab cost <= T possible?  Greedy from z = 0: every slab
    // takes as many granules as fit under T, at least mg, and leaves mg for
    // each slab after it (taking more never hurts the slabs after it).
    auto feasible = [&](double T, std::vector<int64_t> *out) {
        int64_t q = 0;
        if (out) out->assign(1, 0);
        for (int64_t r = 0; r < nranks; ++r) {
            const int64_t lo = q + mg, hi = ng - (nranks - 1 - r) * mg;
            if (lo > hi) return false;
            int64_t e = lo;
            if (r == nranks - 1)
                e = ng;
            else
                while (e < hi && pre[(size_t)e + 1] - pre[(size_t)q] <= T) ++e;
            if (pre[(size_t)e] - pre[(size_t)q] > T) return false;
            if (out) out->push_back(e);
            q = e;
        }
        return true;
    };
    double lo = 0.0, hi = pre[(size_t)ng];   // hi is always feasible
    for (int it = 0; it < 200 && hi - lo > 1e-13 * hi; ++it) {
        const double mid = 0.5 * (lo + hi);
        if (feasible(mid, nullptr)) hi = mid; else lo = mid;
    }
    std::vector<int64_t> g;
    feasible(hi, &g);
    for (int64_t r = 0; r <= nranks; ++r) z_split[r] = g[(size_t)r] * granule;
    return PIC_OK;
}

int pic_get_stage_times(pic_ctx *ctx, double ms[4], int64_t *particle_launches)
{
    if (!ctx || !ms) return PIC_EINVAL;
    for (int i = 0; i < 4; ++i) {
        ms[i] = ctx->stage_ms[i];
        ctx->stage_ms[i] = 0;
    }
    if (particle_launches) *particle_launches = ctx->particle_launches;
    ctx->particle_launches = 0;
    return PIC_OK;
}

int pic_get_launch_count(pic_ctx *ctx, int64_t *launches)
{
    if (!ctx || !launches) return PIC_EINVAL;
    *launches = ctx->launches;
    ctx->launches = 0;
    return PIC_OK;
}

const char *pic_strerror(int code) { return err_names(code); }

const char *pic_last_error(pic_ctx *ctx)
{
    if (!ctx) return "NULL context";
    return ctx->last_error.c_str();
}

void pic_destroy(pic_ctx *ctx)
{
    if (!ctx) return;
    destroy_graphs(ctx);
    for (auto e : ctx->ev_pool) cudaEventDestroy(e);
    if (ctx->comm) {
        NcclApi *api = nccl_api();
        if (api) api->commDestroy(ctx->comm);
    }
    if (ctx->ev_occ) cudaEventDestroy(ctx->ev_occ);
    if (ctx->h_occ) cudaFreeHost(ctx->h_occ);
    if (ctx->ev_fork) cudaEventDestroy(ctx->ev_fork);
    if (ctx->ev_join) cudaEventDestroy(ctx->ev_join);
    if (ctx->st_x) cudaStreamDestroy(ctx->st_x);
    delete ctx;
}

}  // extern "C"
