// handle.cuh -- host-side state of one batched plan (C++ only).
#pragma once

#include <string>
#include <vector>

#include "sgiga_internal.cuh"

namespace sgiga {

void set_error(const std::string& msg);

#define SG_CUDA(call)                                                             \
    do {                                                                          \
        cudaError_t _e = (call);                                                  \
        if (_e != cudaSuccess) {                                                  \
            ::sgiga::set_error(std::string(#call) + ": " + cudaGetErrorString(_e)); \
            return SGIGA_ERR_CUDA;                                                \
        }                                                                         \
    } while (0)

// launch counter that also advances the handle's launch sequence number
struct LaunchCount {
    long long n = 0;
    long long* seq = nullptr;
    LaunchCount& operator++() { ++n; ++*seq; return *this; }
    long long operator++(int) { const long long o = n; ++*this; return o; }
    LaunchCount& operator+=(long long k) { n += k; ++*seq; return *this; }
    LaunchCount& operator=(long long v) { n = v; return *this; }
    operator long long() const { return n; }
};

// Developer / test switches, read ONCE from the environment when a handle
// is created (never on a launch path).  Defaults are the product path.
struct Options {
    bool no_fd = false;             // SGIGA_NO_FD=1: Jacobi-PCG instead of FD-PCG (parity tests)
    bool generic_assembly = false;  // SGIGA_GENERIC_ASSEMBLY=1: runtime-size assembly kernel (parity tests)
    bool no_tma = false;            // SGIGA_NO_TMA=1: cp.async plane copies instead of TMA (parity tests)
    bool no_ktimes = false;         // SGIGA_NO_KTIMES=1: no kernel-group timing events
    bool run_graph = false;         // SGIGA_RUN_GRAPH=1 (and no SGIGA_NO_GRAPH): whole-pass CUDA graphs
    bool no_cluster = false;        // SGIGA_NO_CLUSTER=1: chunked Jacobi-PCG for the small comps (tests)
    bool combine_nosort = false;    // SGIGA_COMBINE_NOSORT=1: no cell sort of the points (tests)
    bool combine_perthread = false; // SGIGA_COMBINE_PERTHREAD=1: per-thread combine kernel (tests)
    bool asm_profile = false;       // SGIGA_ASM_PROFILE=1: block-0 stage cycles to stderr (probe)
    bool asm_pencil = false;        // SGIGA_ASM_PENCIL=1: one-pencil-per-CTA 3-D assembly (parity tests)
    bool no_box_asm = false;        // SGIGA_NO_BOX_ASM=1: box geometries through the tiled / pencil assembly (tests)
    bool no_box_metric = false;     // SGIGA_NO_BOX_METRIC=1: box geometries through the general contraction (k_metric; tests)
    bool no_diag_metric = false;    // SGIGA_NO_DIAG=1: general-metric tiled assembly on box geometries (tests)
    bool fd_profile = false;        // SGIGA_FD_PROFILE=1: FD phase cycles to stderr (probe)
    bool pcg_profile = false;       // SGIGA_PCG_PROFILE=1 (probe)
    bool pcg_trace = false;         // SGIGA_PCG_TRACE=1 (probe)
    static Options from_env();
};

struct Handle {
    int dev = 0;
    Options opt = Options::from_env();
    cudaStream_t stream = nullptr;
    bool own_stream = false;

    // problem
    int d = 0, p = 0, r = 0, q = 0, mu = 1, ncomp = 0, max_level = 0, forcing_id = 0;
    std::vector<int> levels, coefs;
    std::vector<double> gauss_n, gauss_w;
    GeoInfo geo{};
    std::vector<double> geo_knots, geo_hw;

    // component / table / work lists (host mirrors)
    std::vector<CompInfo> comps;
    std::vector<TabInfo> tabs;
    std::vector<int> tab_of;           // [d*(max_level+1)] -> tab index
    std::vector<double> bp_host;       // concatenated breakpoints
    std::vector<Pencil> pencils;
    std::vector<Block2> blocks2;       // 2-D assembly blocks (k_assembly2d.cu)
    Block2* d_blocks2 = nullptr;
    std::vector<Chunk> chunks;
    std::vector<int> small_comps, large_comps;
    std::vector<int> slotoff;          // per-component slot column offsets
    int* d_slotoff = nullptr;
    int64_t total_qp = 0, total_rows = 0, total_vec = 0, total_slots = 0, total_dofs = 0;
    int64_t total_knots = 0, total_tabvals = 0, total_tabqp = 0;
    int max_slots_comp = 0;

    // device buffers
    CompInfo* d_comps = nullptr;
    TabInfo* d_tabs = nullptr;
    GeoInfo* d_geo = nullptr;
    Pencil* d_pencils = nullptr;
    Chunk* d_chunks = nullptr;
    int* d_small = nullptr;
    int* d_large = nullptr;
    double* d_bp = nullptr;
    double* d_knots = nullptr;
    double* d_gauss = nullptr;   // nodes [q], weights [q]
    double* d_tabvals = nullptr;
    double* d_qx = nullptr;      // xi at table quad points
    double* d_qw = nullptr;      // h * w_g
    double* d_geob = nullptr;    // geometry basis at table quad points
    int* d_geofirst = nullptr;   // first active geometry function
    double* d_geo_knots = nullptr;
    double* d_geo_hw = nullptr;
    double* d_G = nullptr;       // metric (ncg comps) + load per qp
    double* d_hostf = nullptr;   // host forcing densities (SGIGA_FORCING_HOST)
    double* d_xphys = nullptr;   // physical qp coordinates (host forcing only)
    double* d_stencil = nullptr;
    double* d_rhs = nullptr;
    double* d_dinv = nullptr;
    double* d_x = nullptr;
    double* d_r = nullptr;
    double* d_z = nullptr;
    double* d_p = nullptr;
    double* d_q = nullptr;
    double* d_q2 = nullptr;      // second direction buffer (PCG parity)
    double* d_coef = nullptr;    // full coefficients, reference C order
    CgState* d_cg = nullptr;
    double* d_part = nullptr;    // per-chunk partial sums [3*nchunks]
    int* d_err = nullptr;
    int* d_active_count = nullptr;
    int* d_alist = nullptr;      // compacted active chunk list (large-path PCG)
    double* d_relres = nullptr;
    // FD preconditioner (k_fd.cu): per-table factor offsets (shared between
    // tables with the same knot vector), the tables to factor, the comps
    std::vector<int> fd_comps, fd_uniq;
    std::vector<int64_t> fd_uoff, fd_loff;
    int64_t fd_u_total = 0, fd_l_total = 0;
    int* d_fdlist = nullptr;
    int* d_fd_uniq = nullptr;
    int64_t* d_fd_uoff = nullptr;
    int64_t* d_fd_loff = nullptr;
    double* d_fdU = nullptr;
    double* d_fdL = nullptr;
    // whole-GPU FD-PCG comps (k_pcg_grid.cu): large components, every axis FD
    std::vector<int> fdg_comps;
    int* d_fdg_list = nullptr;
    double* d_fdg_part = nullptr;            // [2][FDG_MAX_CTAS] per-CTA partial sums
    double* d_fdg_ckpart = nullptr;          // [n_fdg][MAXD][256] chunk partials of their c_k
    // line-FD comps (one long axis; k_pcg_fdl): per-comp offset into d_fdl
    // (stream-axis K / M bands + one banded Cholesky factor per line)
    std::vector<int> fdl_comps;
    std::vector<int64_t> fdl_off;
    int64_t fdl_total = 0;
    int* d_fdl_list = nullptr;
    int64_t* d_fdl_off = nullptr;
    double* d_fdl = nullptr;
    double* d_ck = nullptr;                  // [ncomp][MAXD] FD metric scales c_k (k_fd_metric_scale)
    unsigned* d_ticket = nullptr;            // last-CTA ticket of the status-fused combine (kept zero)
    std::vector<double> knots_host;          // open knot vectors (host-built, uploaded once)
    std::vector<int> mcomp;                  // component of k_metric's CTA b (first point b * 256)
    int* d_mcomp = nullptr;                  // k_metric: component of each 256-point CTA
    cudaStream_t stream2 = nullptr;          // side stream: the eigen kernel overlaps assembly
    cudaEvent_t fd_fork = nullptr, fd_join = nullptr, fd_metric = nullptr;
    cudaEvent_t pcg_fork = nullptr, pcg_join = nullptr;   // FD-PCG beside the line-FD PCG
    bool fd_pending = false;                 // fd_join not yet waited on by the main stream
    // combine point sort on its own side stream (sgiga_run: forked before the
    // assembly, joined before the combine kernel)
    cudaStream_t stream3 = nullptr;
    cudaEvent_t cs_fork = nullptr, cs_join = nullptr;
    bool cs_pending = false, cs_ready = false;
    int64_t run_npts = 0;          // points of the last enqueued sgiga_run pass
    int* d_cperm = nullptr;        // combine: cell-order permutation of the points
    size_t cperm_cap = 0;
    int* d_chist = nullptr;        // combine: cell histogram / cursors (zeroed by every sort)
    double* d_spts = nullptr;      // staging of host points (sgiga_run / _combine_points), per handle
    size_t spts_cap = 0;
    double* d_sout = nullptr;      // staging of the values read back to the host, per handle
    size_t sout_cap = 0;
    int* h_pinned_flag = nullptr;  // pinned host mirror of the active count
    int* h_err = nullptr;          // mapped pinned mirrors read after the one sync of a call
    CgState* h_cg = nullptr;
    double* h_rel = nullptr;
    int* h_sticky = nullptr;       // failure word OR-ed by every pass's status writer (mapped)
    int* dh_sticky = nullptr;
    int passes_pending = 0;        // passes enqueued since the last verdict
    int* dh_err = nullptr;         // ... and their device-side addresses
    CgState* dh_cg = nullptr;
    double* dh_rel = nullptr;

    // state
    bool tables_ready = false, density_ready = false, assembled = false, solved = false,
         have_coefs = false;
    // timing marks: slots 0..13 = kernel-group start/stop pairs
    // (sgiga_kernel_times), 14..19 = phase boundaries (sgiga_phase_stats).
    // A mark with no launch since the previous mark reuses that event, so a
    // chain of adjacent boundaries costs one event record, not several.
    static constexpr int NEV = 20, PHASE_EV = 14;
    cudaEvent_t evp[NEV] = {};
    int alias[NEV] = {};
    int last_mark = -1;
    long long last_seq = -1;
    long long seq = 0;            // bumped by every counted launch
    bool kran[7] = {false, false, false, false, false, false, false};
    float ms[3] = {0, 0, 0};
    LaunchCount launches[3] = {{0, &seq}, {0, &seq}, {0, &seq}};
    std::vector<int> iters;
    bool force_generic_assembly = false;   // SGIGA_GENERIC_ASSEMBLY=1 (parity cross-check)
    int asm_seg = 0;                       // stream-axis segment length of the pencils
    int n_pencils_other = 0;               // pencils of the components the tiled kernel does not take (first)
    void* d_tmaps = nullptr;               // per-component CUtensorMap of d_G (TMA plane copies)
    int tmaps_state = 0;                   // 0 = not built, 1 = ready, -1 = unavailable
    // tiled 3-D assembly (k_assembly_tile.cu): tiles, per-component tensor
    // maps with the tile's window box, dynamic shared memory of the launch
    std::vector<Tile3> tiles3;
    Tile3* d_tiles3 = nullptr;
    void* d_tmaps3 = nullptr;
    int tiles3_state = 0;                  // 0 = not built, 1 = ready, -1 = not applicable
    size_t tiles3_smem = 0;
    double tiles3_flops = 0.0;             // FP64 operations one tiled-assembly launch executes
    bool tiles3_dg = false;                // diagonal-metric instantiation (axis-aligned box geometry)
    // Kronecker assembly of box geometries (k_assembly_box.cu)
    int box_state = 0;                     // 0 = not built, 1 = ready, -1 = not applicable
    double* d_box1d = nullptr;             // 1-D mass / stiffness bands per knot vector
    int64_t* d_box_tcum = nullptr;         // band offsets (entries) per knot vector
    void* d_box_stage = nullptr;           // load sum-factorisation stages (3 per component)
    void* d_box_work = nullptr;            // their CTA work lists
    double* d_box_x1 = nullptr;            // stage buffers
    double* d_box_x2 = nullptr;
    int box_nwork[3] = {0, 0, 0};
    int64_t box_tab_total = 0;
    bool stencil_zeroed = false;           // the stencil's structural zeros are in place (set once per layout)
    bool metric_offdiag_zeroed = false;    // the metric's exactly-zero off-diagonal entries are in place (box geometry)
    bool asm_tiled = false;                // the last assembly ran k_assemble_tile
    bool small_checked = false;            // small comps' true residual came from the cluster PCG

    // whole-run CUDA graph (sgiga_run): captured on the second call with the
    // same arguments, replayed while they and the work lists stay the same
    bool capturing = false, graph_broken = false;
    cudaGraphExec_t run_exec = nullptr;
    struct RunKey {
        double rtol = 0.0;
        int maxit = 0, warm = 0;
        const double* dp = nullptr;
        const double* hp = nullptr;   // pinned host source of the points (uploaded inside the pass)
        double* dout = nullptr;
        int64_t npts = -1;
    } rkey;
    long long run_launches[3] = {0, 0, 0};
    bool run_kran[7] = {false, false, false, false, false, false, false};
    int run_alias[NEV] = {};
    void drop_run_graph() {
        if (run_exec) cudaGraphExecDestroy(run_exec);
        run_exec = nullptr;
        rkey = RunKey{};
    }

    // event record that is also a timing node when the stream is captured
    cudaError_t rec(cudaEvent_t e) {
        return capturing ? cudaEventRecordWithFlags(e, stream, cudaEventRecordExternal)
                         : cudaEventRecord(e, stream);
    }
    void mark(int slot) {
        if (last_mark >= 0 && last_seq == seq) { alias[slot] = last_mark; return; }
        rec(evp[slot]);
        alias[slot] = slot;
        last_mark = slot;
        last_seq = seq;
    }
    void begin_call() { last_mark = -1; }   // never alias an event of an earlier call
    cudaError_t elapsed(float* out, int a, int b) const {
        return cudaEventElapsedTime(out, evp[alias[a]], evp[alias[b]]);
    }
    bool ktimes = true;   // kernel-group events (SGIGA_NO_KTIMES=1 turns them off)
    void kstart(int g) { if (ktimes) { mark(2 * g); kran[g] = true; } }
    void kstop(int g) { if (ktimes) mark(2 * g + 1); }
    void pmark(int i) { mark(PHASE_EV + i); }
    int ncg() const { return d * (d + 1) / 2; }   // symmetric metric entries
    int nG() const { return ncg() + 1; }           // + load
};

// the tiled 3-D assembly (k_assembly_tile.cu) can serve this plan (d = 3,
// maximal regularity, q = p + 1, degree 3 or 4); the per-component choice
// is CompInfo::tile3 (components with at least TILE3_MIN_ELEMENTS elements)
bool tile3_eligible(const Handle* h);
// axis-aligned box geometry: the metric's off-diagonal entries are exact zeros
bool metric_diagonal(const Handle* h);
// box geometry constants: corner c0, edge lengths L, g_k = det / L_k^2, det
void box_constants(const Handle* h, double* c0, double* L, double* g, double* det);
bool box_assembly_eligible(const Handle* h);
bool box_assembly_ready(Handle* h);   // eligible and its tables built (the pass will run it)
void free_box(Handle* h);
constexpr double TILE3_MIN_ELEMENTS = 512.0;

// symmetric index of (m, n) in the packed metric (row-major upper triangle)
__host__ __device__ inline int sym_index(int d, int m, int n) {
    if (m > n) { int t = m; m = n; n = t; }
    // rows: m=0: n=0..d-1 ; m=1: n=1..d-1 ; ...
    return m * d - (m * (m - 1)) / 2 + (n - m);
}

}  // namespace sgiga
