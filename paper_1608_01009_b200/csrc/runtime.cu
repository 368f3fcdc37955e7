// runtime.cu -- the C ABI of libpic.so (include/pic.h): validation,
// workspace carving, the per-step launch schedule, CUDA graph capture,
// stage timing and the sticky device error word.
//
// Per step n:
//   a1  n % K == 0: stable sort A -> B per species (sort.cu)
//   a2-a6 particle kernel per species, input B on a sort step else A,
//       output A (in place), deposit into J_cur
//   a7  B half, E full (+ J fold, zero J_next), B half (fields.cu)
//   swap J_cur / J_next
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/pic.h"
#include "kernels.cuh"

using namespace pic;

namespace {

constexpr size_t kAlign = 256;
inline size_t align_up(size_t v) { return (v + kAlign - 1) / kAlign * kAlign; }

struct Layout {
    GridDev g{};
    int64_t ncells = 0, n_sc = 0;
    int64_t cap[PIC_MAX_SPECIES] = {};
    int64_t cap_max = 0;
    size_t off_eb = 0, off_j[2] = {}, off_sp[PIC_MAX_SPECIES][2] = {}, off_scoff[PIC_MAX_SPECIES] = {};
    size_t off_key = 0, off_slot = 0, off_perm_tmp = 0, off_perm = 0, off_count = 0, off_start = 0,
           off_bsums = 0, off_err = 0, off_stat = 0;
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
    if (c->nz % c->nranks) return "nz must be divisible by nranks";
    if (c->supercell < 1) return "supercell must be >= 1";
    const int64_t nzl = c->nz / c->nranks;
    if (c->nx % c->supercell || c->ny % c->supercell || nzl % c->supercell)
        return "supercell must divide nx, ny and nz/nranks";
    if (c->sort_every < 0) return "sort_every must be >= 0";
    if (c->nx * c->ny * nzl >= (int64_t(1) << 31)) return "local grid too large";
    if (c->nranks > 1) return "nranks > 1: z-slab exchange not built in this version";
    return "";
}

Layout make_layout(const pic_config *c)
{
    Layout L;
    GridDev &g = L.g;
    g.nx = (int)c->nx;
    g.ny = (int)c->ny;
    g.nz = (int)(c->nz / c->nranks);
    g.nz_global = (int)c->nz;
    g.k0 = (int)(c->rank * g.nz);
    g.X = g.nx + 2 * kGhost;
    g.X += g.X & 1;   // 16-byte row pitch
    g.Y = g.ny + 2 * kGhost;
    g.Z = g.nz + 2 * kGhost;
    g.cs = (int64_t)g.X * g.Y * g.Z;
    g.cs += (g.cs & 1);
    g.dx = c->dx; g.dy = c->dy; g.dz = c->dz;
    g.inv_dx = 1.0 / c->dx; g.inv_dy = 1.0 / c->dy; g.inv_dz = 1.0 / c->dz;
    g.dt = c->dt; g.c = c->c;
    g.Lx = c->nx * c->dx; g.Ly = c->ny * c->dy; g.Lz = c->nz * c->dz;
    g.S = (int)c->supercell;
    g.nsx = g.nx / g.S; g.nsy = g.ny / g.S; g.nsz = g.nz / g.S;
    g.periodic_z_local = (c->nranks == 1);
    L.ncells = (int64_t)g.nx * g.ny * g.nz;
    L.n_sc = (int64_t)g.nsx * g.nsy * g.nsz;
    size_t o = 0;
    L.off_eb = o; o = align_up(o + sizeof(double) * 6 * (size_t)g.cs);
    for (int b = 0; b < 2; ++b) { L.off_j[b] = o; o = align_up(o + sizeof(double) * 3 * (size_t)g.cs); }
    for (int s = 0; s < c->n_species; ++s) {
        L.cap[s] = c->capacity[s];
        L.cap_max = std::max(L.cap_max, L.cap[s]);
        for (int b = 0; b < 2; ++b) {
            L.off_sp[s][b] = o;
            o = align_up(o + (sizeof(double) * 6 + sizeof(uint64_t)) * (size_t)L.cap[s] + 6 * kAlign);
        }
        L.off_scoff[s] = o; o = align_up(o + sizeof(int64_t) * (size_t)(L.n_sc + 1));
    }
    const size_t capm = (size_t)std::max<int64_t>(L.cap_max, 1);
    L.off_key = o; o = align_up(o + 4 * capm);
    L.off_slot = o; o = align_up(o + 4 * capm);
    L.off_perm_tmp = o; o = align_up(o + 4 * capm);
    L.off_perm = o; o = align_up(o + 4 * capm);
    L.off_count = o; o = align_up(o + 4 * (size_t)(L.ncells + 1));
    L.off_start = o; o = align_up(o + 4 * (size_t)(L.ncells + 1));
    L.off_bsums = o; o = align_up(o + 4 * scan_block_count(L.ncells + 1));
    L.off_err = o; o = align_up(o + 64);
    L.off_stat = o; o = align_up(o + 2 * PIC_MAX_SPECIES * sizeof(unsigned));
    L.total = o;
    return L;
}

ParticlesDev carve_particles(char *base, size_t off, int64_t cap)
{
    ParticlesDev p;
    const size_t col = align_up(sizeof(double) * (size_t)cap);
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

}  // namespace

struct pic_ctx {
    pic_config cfg{};
    Layout L;
    char *ws = nullptr;
    cudaStream_t st = nullptr;
    double *EB = nullptr;
    double *J[2] = {nullptr, nullptr};
    int jcur = 0;              // J buffer receiving the next deposit
    int jlast = 1;             // J buffer holding J^{n-1/2}
    ParticlesDev A[PIC_MAX_SPECIES], B[PIC_MAX_SPECIES];
    int64_t *sc_off[PIC_MAX_SPECIES] = {};
    int64_t count[PIC_MAX_SPECIES] = {};
    SortScratch sort{};
    unsigned *err = nullptr;
    unsigned *u2max[2] = {nullptr, nullptr};   // [parity][species], see SpeciesDev
    int64_t step_index = 0;
    bool use_tile = false;     // fused supercell kernel (else the naive kernel)
    CUtensorMap eb_map;        // TMA descriptor of the padded E/B array [6][Z][Y][X]
    int num_sms = 148;
    std::string last_error;
    // graphs keyed by (sort_now, jcur)
    cudaGraphExec_t graph[2][2] = {{nullptr, nullptr}, {nullptr, nullptr}};
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

// Enqueue one full step; returns the number of kernel launches enqueued.
int enqueue_step(pic_ctx *ctx, bool sort_now, int jcur, bool profile)
{
    const Layout &L = ctx->L;
    const GridDev &g = L.g;
    int launches = 0;
    if (sort_now) {
        StageMark m(ctx, 0, profile);
        for (int s = 0; s < ctx->cfg.n_species; ++s)
            sort_particles(g, ctx->A[s], ctx->B[s], ctx->count[s], ctx->sort, ctx->sc_off[s],
                           ctx->err, ctx->st, &launches);
    }
    {
        StageMark m(ctx, 1, profile);
        // u^2 bounds: this step reads parity jcur, writes parity 1 - jcur
        cudaMemsetAsync(ctx->u2max[1 - jcur], 0, PIC_MAX_SPECIES * sizeof(unsigned), ctx->st);
        for (int s = 0; s < ctx->cfg.n_species; ++s) {
            if (ctx->count[s] == 0) continue;
            SpeciesDev sp;
            sp.qw = ctx->cfg.q[s] * ctx->cfg.w[s];
            sp.h = ctx->cfg.q[s] * g.dt / (2.0 * ctx->cfg.m[s] * g.c);
            sp.u2max_in = ctx->u2max[jcur] + s;
            sp.u2max_out = ctx->u2max[1 - jcur] + s;
            const ParticlesDev &in = sort_now ? ctx->B[s] : ctx->A[s];
            if (ctx->use_tile)
                launch_push_tile(ctx->eb_map, g, ctx->EB, ctx->J[jcur], in, ctx->A[s], ctx->sc_off[s],
                                 sp, sort_now, ctx->err, ctx->num_sms, ctx->st);
            else
                launch_push_naive(g, ctx->EB, ctx->J[jcur], in, ctx->A[s], ctx->count[s], sp,
                                  sort_now, ctx->err, ctx->st);
            ++launches;
            if (profile) ctx->particle_launches++;
        }
    }
    {
        StageMark m(ctx, 2, profile);
        launch_b_half(g, ctx->EB, ctx->st);
        launch_e_full(g, ctx->EB, ctx->J[jcur], ctx->J[1 - jcur], ctx->st);
        launch_b_half(g, ctx->EB, ctx->st);
        launches += 3;
    }
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
    if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaStreamEndCapture");
    e = cudaGraphInstantiate(&ctx->graph[sort_now][jcur], graph, 0);
    cudaGraphDestroy(graph);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaGraphInstantiate");
    ctx->graph_launches[sort_now][jcur] = n;
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
    tile_box(g.S, bx);
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

int check_device_error(pic_ctx *ctx)
{
    unsigned h = 0;
    PIC_CUDA(ctx, cudaMemcpyAsync(&h, ctx->err, sizeof(unsigned), cudaMemcpyDeviceToHost, ctx->st));
    PIC_CUDA(ctx, cudaStreamSynchronize(ctx->st));
    if (h & kErrNonFinite) return fail(ctx, PIC_ENONFINITE, "non-finite particle state");
    if (h & kErrDisplacement) return fail(ctx, PIC_EDISPLACEMENT, "displacement >= 1 cell");
    if (h & kErrRange) return fail(ctx, PIC_EINVAL, "particle position outside the domain");
    if (h & kErrCapacity) return fail(ctx, PIC_ECAPACITY, "device capacity exceeded");
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
    ctx->EB = (double *)(ctx->ws + L.off_eb);
    ctx->J[0] = (double *)(ctx->ws + L.off_j[0]);
    ctx->J[1] = (double *)(ctx->ws + L.off_j[1]);
    for (int s = 0; s < cfg->n_species; ++s) {
        ctx->A[s] = carve_particles(ctx->ws, L.off_sp[s][0], L.cap[s]);
        ctx->B[s] = carve_particles(ctx->ws, L.off_sp[s][1], L.cap[s]);
        ctx->sc_off[s] = (int64_t *)(ctx->ws + L.off_scoff[s]);
    }
    ctx->sort.key = (uint32_t *)(ctx->ws + L.off_key);
    ctx->sort.slot = (uint32_t *)(ctx->ws + L.off_slot);
    ctx->sort.perm_tmp = (uint32_t *)(ctx->ws + L.off_perm_tmp);
    ctx->sort.perm = (uint32_t *)(ctx->ws + L.off_perm);
    ctx->sort.count = (uint32_t *)(ctx->ws + L.off_count);
    ctx->sort.start = (uint32_t *)(ctx->ws + L.off_start);
    ctx->sort.block_sums = (uint32_t *)(ctx->ws + L.off_bsums);
    ctx->err = (unsigned *)(ctx->ws + L.off_err);
    ctx->u2max[0] = (unsigned *)(ctx->ws + L.off_stat);
    ctx->u2max[1] = ctx->u2max[0] + PIC_MAX_SPECIES;
    ctx->use_tile = !(cfg->flags & PIC_FLAG_NAIVE) && tile_supported((int)cfg->supercell);
    configure_tile_kernels();
    {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, dev);
        const char *pe = getenv("PIC_TILE_PERSISTENT");   // tuning knob: "0" = one CTA per supercell
        if (pe && pe[0] == '0') ctx->num_sms = 0;
    }
    if (ctx->use_tile && encode_eb_map(ctx) != PIC_OK) {
        delete ctx;
        return PIC_ECUDA;
    }
    // zero fields, offsets and the error word (particle arrays stay garbage until set)
    cudaError_t e = cudaMemsetAsync(ctx->ws, 0, L.off_sp[0][0], ctx->st);
    for (int s = 0; e == cudaSuccess && s < cfg->n_species; ++s)
        e = cudaMemsetAsync(ctx->sc_off[s], 0, sizeof(int64_t) * (size_t)(L.n_sc + 1), ctx->st);
    if (e == cudaSuccess) e = cudaMemsetAsync(ctx->err, 0, 64, ctx->st);
    if (e == cudaSuccess) e = cudaMemsetAsync(ctx->u2max[0], 0, 2 * PIC_MAX_SPECIES * sizeof(unsigned), ctx->st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->st);
    if (e != cudaSuccess) {
        delete ctx;
        return PIC_ECUDA;
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
    if (n > ctx->L.cap[species]) return fail(ctx, PIC_ECAPACITY, "n exceeds capacity");
    const GridDev &g = ctx->L.g;
    for (int64_t p = 0; p < n; ++p) {
        if (!(x[p] >= 0.0 && x[p] < g.Lx && y[p] >= 0.0 && y[p] < g.Ly && z[p] >= 0.0 && z[p] < g.Lz))
            return fail(ctx, PIC_EINVAL, "particle position outside [0, L)");
    }
    const ParticlesDev &Bs = ctx->B[species];
    const size_t bytes = sizeof(double) * (size_t)n;
    const double *src[6] = {x, y, z, ux, uy, uz};
    double *dst[6] = {Bs.x, Bs.y, Bs.z, Bs.ux, Bs.uy, Bs.uz};
    for (int c = 0; c < 6 && n > 0; ++c)
        PIC_CUDA(ctx, cudaMemcpyAsync(dst[c], src[c], bytes, cudaMemcpyHostToDevice, ctx->st));
    if (n > 0)
        PIC_CUDA(ctx, cudaMemcpyAsync(Bs.id, id, sizeof(uint64_t) * (size_t)n, cudaMemcpyHostToDevice, ctx->st));
    ctx->count[species] = n;
    int launches = 0;
    sort_particles(g, Bs, ctx->A[species], n, ctx->sort, ctx->sc_off[species], ctx->err, ctx->st,
                   &launches);
    launch_u2max(ctx->A[species], n, ctx->u2max[ctx->jcur] + species, ctx->st);
    ++launches;
    ctx->launches += launches;
    PIC_CUDA(ctx, cudaGetLastError());
    destroy_graphs(ctx);
    return check_device_error(ctx);
}

int pic_set_fields(pic_ctx *ctx, const double *f)
{
    if (!ctx || !f) return PIC_EINVAL;
    const GridDev &g = ctx->L.g;
    for (int c = 0; c < 6; ++c) {
        cudaMemcpy3DParms p = {};
        p.srcPtr = make_cudaPitchedPtr((void *)(f + (size_t)c * g.nx * g.ny * g.nz),
                                       sizeof(double) * g.nx, g.nx, g.ny);
        p.dstPtr = make_cudaPitchedPtr(ctx->EB + c * g.cs, sizeof(double) * g.X, g.X, g.Y);
        p.dstPos = make_cudaPos(sizeof(double) * kGhost, kGhost, kGhost);
        p.extent = make_cudaExtent(sizeof(double) * g.nx, g.ny, g.nz);
        p.kind = cudaMemcpyHostToDevice;
        PIC_CUDA(ctx, cudaMemcpy3DAsync(&p, ctx->st));
    }
    launch_fill_ghosts(g, ctx->EB, 6, ctx->st);
    ctx->launches += 1;
    PIC_CUDA(ctx, cudaGetLastError());
    PIC_CUDA(ctx, cudaStreamSynchronize(ctx->st));
    return PIC_OK;
}

int pic_get_fields(pic_ctx *ctx, double *f)
{
    if (!ctx || !f) return PIC_EINVAL;
    const GridDev &g = ctx->L.g;
    for (int c = 0; c < 9; ++c) {
        const double *srcbase = c < 6 ? ctx->EB + c * g.cs : ctx->J[ctx->jlast] + (c - 6) * g.cs;
        cudaMemcpy3DParms p = {};
        p.srcPtr = make_cudaPitchedPtr((void *)srcbase, sizeof(double) * g.X, g.X, g.Y);
        p.srcPos = make_cudaPos(sizeof(double) * kGhost, kGhost, kGhost);
        p.dstPtr = make_cudaPitchedPtr(f + (size_t)c * g.nx * g.ny * g.nz, sizeof(double) * g.nx,
                                       g.nx, g.ny);
        p.extent = make_cudaExtent(sizeof(double) * g.nx, g.ny, g.nz);
        p.kind = cudaMemcpyDeviceToHost;
        PIC_CUDA(ctx, cudaMemcpy3DAsync(&p, ctx->st));
    }
    PIC_CUDA(ctx, cudaStreamSynchronize(ctx->st));
    return PIC_OK;
}

int pic_get_particles(pic_ctx *ctx, int species, int64_t *n_inout, double *x, double *y, double *z,
                      double *ux, double *uy, double *uz, uint64_t *id)
{
    if (!ctx || !n_inout) return PIC_EINVAL;
    if (species < 0 || species >= ctx->cfg.n_species) return fail(ctx, PIC_EINVAL, "bad species");
    const int64_t n = ctx->count[species];
    const int64_t capacity = *n_inout;
    *n_inout = n;
    if (capacity < n) return fail(ctx, PIC_ECAPACITY, "output arrays too small");
    const ParticlesDev &A = ctx->A[species];
    const double *src[6] = {A.x, A.y, A.z, A.ux, A.uy, A.uz};
    double *dst[6] = {x, y, z, ux, uy, uz};
    for (int c = 0; c < 6 && n > 0; ++c)
        if (dst[c])
            PIC_CUDA(ctx, cudaMemcpyAsync(dst[c], src[c], sizeof(double) * (size_t)n,
                                          cudaMemcpyDeviceToHost, ctx->st));
    if (id && n > 0)
        PIC_CUDA(ctx, cudaMemcpyAsync(id, A.id, sizeof(uint64_t) * (size_t)n, cudaMemcpyDeviceToHost, ctx->st));
    PIC_CUDA(ctx, cudaStreamSynchronize(ctx->st));
    return PIC_OK;
}

int pic_get_count(pic_ctx *ctx, int species, int64_t *n)
{
    if (!ctx || !n || species < 0 || species >= ctx->cfg.n_species) return PIC_EINVAL;
    *n = ctx->count[species];
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
    const int64_t K = ctx->cfg.sort_every;
    const bool profile = (ctx->cfg.flags & PIC_FLAG_PROFILE) != 0;
    const bool use_graph = !profile && !(ctx->cfg.flags & PIC_FLAG_NO_GRAPH) && ctx->st != nullptr;
    for (int64_t s = 0; s < nsteps; ++s) {
        const bool sort_now = K > 0 && (ctx->step_index % K) == 0;
        const int jc = ctx->jcur;
        if (use_graph) {
            if (!ctx->graphs_valid) {
                destroy_graphs(ctx);
                ctx->graphs_valid = true;
            }
            if (!ctx->graph[sort_now][jc]) {
                int rc = build_graph(ctx, sort_now, jc);
                if (rc != PIC_OK) return rc;
            }
            PIC_CUDA(ctx, cudaGraphLaunch(ctx->graph[sort_now][jc], ctx->st));
            ctx->launches += ctx->graph_launches[sort_now][jc];
        } else {
            ctx->launches += enqueue_step(ctx, sort_now, jc, profile);
            PIC_CUDA(ctx, cudaGetLastError());
        }
        ctx->jlast = jc;
        ctx->jcur = 1 - jc;
        ctx->step_index++;
    }
    int rc = check_device_error(ctx);
    if (profile) {
        for (auto &m : ctx->ev_marks) {
            float ms = 0.f;
            cudaEventElapsedTime(&ms, m.second.first, m.second.second);
            ctx->stage_ms[m.first] += ms;
        }
        ctx->ev_marks.clear();
        ctx->ev_used = 0;
    }
    return rc;
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
    delete ctx;
}

}  // extern "C"
