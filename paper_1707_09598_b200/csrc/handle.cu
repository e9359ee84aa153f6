// handle.cu -- C ABI of libsgiga: descriptor validation, the batch-wide
// component table, device allocation, phase orchestration and exports.
//
// Reference boundary: scheduler.run_plan (scheduler.py:74-96) ->
// combination.solve_component (combination.py:183-200) per component;
// here a whole plan is one handle and every phase is one batched launch.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "handle.cuh"

namespace sgiga {

static thread_local std::string g_last_error;
void set_error(const std::string& msg) { g_last_error = msg; }

static bool env_on(const char* name) {
    const char* e = getenv(name);
    return e && e[0] == '1';
}
Options Options::from_env() {
    Options o;
    o.no_fd = env_on("SGIGA_NO_FD");
    o.generic_assembly = env_on("SGIGA_GENERIC_ASSEMBLY");
    o.no_tma = env_on("SGIGA_NO_TMA");
    o.no_ktimes = env_on("SGIGA_NO_KTIMES");
    o.run_graph = env_on("SGIGA_RUN_GRAPH") && !env_on("SGIGA_NO_GRAPH");
    o.no_cluster = env_on("SGIGA_NO_CLUSTER");
    o.combine_nosort = env_on("SGIGA_COMBINE_NOSORT");
    o.combine_perthread = env_on("SGIGA_COMBINE_PERTHREAD");
    o.asm_profile = env_on("SGIGA_ASM_PROFILE");
    o.asm_pencil = env_on("SGIGA_ASM_PENCIL");
    o.no_diag_metric = env_on("SGIGA_NO_DIAG");
    o.no_box_metric = env_on("SGIGA_NO_BOX_METRIC");
    o.no_box_asm = env_on("SGIGA_NO_BOX_ASM");
    o.fd_profile = env_on("SGIGA_FD_PROFILE");
    o.pcg_profile = env_on("SGIGA_PCG_PROFILE");
    o.pcg_trace = env_on("SGIGA_PCG_TRACE");
    return o;
}

size_t assembly_smem_bytes(const Handle* h);

// cumulative tables stored behind d_gauss: [2q] gauss, then
// tab_qp_cum [ntab+1], comp_qp_cum [ncomp+1], comp_dof_cum [ncomp+1]
static int64_t* cum_base(Handle* h) {
    return reinterpret_cast<int64_t*>(h->d_gauss + 2 * h->q);
}
int64_t* tab_qp_cum_ptr(Handle* h) { return cum_base(h); }
int64_t* comp_qp_cum_ptr(Handle* h) { return cum_base(h) + h->tabs.size() + 1; }
int64_t* comp_dof_cum_ptr(Handle* h) { return comp_qp_cum_ptr(h) + h->ncomp + 1; }

template <typename T>
static cudaError_t dalloc(T** p, size_t n) {
    return cudaMalloc(reinterpret_cast<void**>(p), std::max<size_t>(n, 1) * sizeof(T));
}

static void free_all(Handle* h) {
    void* ptrs[] = {h->d_comps, h->d_tabs, h->d_geo, h->d_pencils, h->d_chunks, h->d_small,
                    h->d_large, h->d_bp, h->d_knots, h->d_gauss, h->d_tabvals, h->d_qx,
                    h->d_qw, h->d_geob, h->d_geofirst, h->d_geo_knots, h->d_geo_hw, h->d_G,
                    h->d_hostf, h->d_xphys, h->d_stencil, h->d_rhs, h->d_dinv, h->d_x,
                    h->d_r, h->d_z, h->d_p, h->d_q, h->d_q2, h->d_coef, h->d_cg, h->d_part, h->d_err,
                    h->d_active_count, h->d_relres, h->d_slotoff, h->d_alist, h->d_cperm, h->d_chist,
                    h->d_fdlist, h->d_fd_uniq, h->d_fd_uoff, h->d_fd_loff, h->d_fdU, h->d_fdL, h->d_tmaps,
                    h->d_fdl_list, h->d_fdl_off, h->d_fdl, h->d_ck, h->d_ticket, h->d_mcomp,
                    h->d_spts, h->d_sout, h->d_blocks2, h->d_fdg_list, h->d_fdg_part, h->d_fdg_ckpart,
                    h->d_tiles3, h->d_tmaps3};
    for (void* p : ptrs)
        if (p) cudaFree(p);
    free_box(h);
    void* hptrs[] = {h->h_pinned_flag, h->h_err, h->h_cg, h->h_rel, h->h_sticky};
    for (void* p : hptrs)
        if (p) cudaFreeHost(p);
    for (auto& e : h->evp)
        if (e) cudaEventDestroy(e);
    if (h->fd_fork) cudaEventDestroy(h->fd_fork);
    if (h->fd_join) cudaEventDestroy(h->fd_join);
    if (h->fd_metric) cudaEventDestroy(h->fd_metric);
    if (h->pcg_fork) cudaEventDestroy(h->pcg_fork);
    if (h->pcg_join) cudaEventDestroy(h->pcg_join);
    if (h->stream2) cudaStreamDestroy(h->stream2);
    if (h->cs_fork) cudaEventDestroy(h->cs_fork);
    if (h->cs_join) cudaEventDestroy(h->cs_join);
    if (h->stream3) cudaStreamDestroy(h->stream3);
    if (h->run_exec) cudaGraphExecDestroy(h->run_exec);
    if (h->own_stream && h->stream) cudaStreamDestroy(h->stream);
}

// ---------------------------------------------------------------------------
// descriptor -> component table (host)
// ---------------------------------------------------------------------------
// k_assembly2d walks the shorter axis of a 2-D component (few, full-width
// barrier intervals) and tiles the longer one
static inline int walk2d_axis(const CompInfo& C) { return C.m[0] <= C.m[1] ? 0 : 1; }

static int build_tables(Handle* h, const sgiga_problem_desc* D) {
    const int d = D->d, p = D->degree;
    if (d < 1 || d > 3) { set_error("dimension must be 1, 2 or 3"); return SGIGA_ERR_VALUE; }
    if (p < 1 || p + 1 > PMAX) { set_error("device path supports degree 1..4"); return SGIGA_ERR_VALUE; }
    if (D->regularity < 0 || D->regularity > p - 1) {
        set_error("device path supports regularity in [0, degree-1]");
        return SGIGA_ERR_VALUE;
    }
    if (D->quad_points < 1 || D->quad_points > QMAX) {
        set_error("quadrature points per direction must be in [1, 10]");
        return SGIGA_ERR_VALUE;
    }
    if (D->n_comp < 1) { set_error("a combination plan needs at least one term"); return SGIGA_ERR_VALUE; }
    if (D->max_level < 0 || D->max_level > 30) { set_error("max_level out of range"); return SGIGA_ERR_VALUE; }
    h->d = d; h->p = p; h->r = D->regularity; h->q = D->quad_points; h->mu = p - D->regularity;
    h->ncomp = D->n_comp; h->max_level = D->max_level; h->forcing_id = D->forcing_id;
    if (h->forcing_id < SGIGA_FORCING_HOST || h->forcing_id > SGIGA_FORCING_LSHAPE) {
        set_error("unknown forcing id");
        return SGIGA_ERR_VALUE;
    }
    h->levels.assign(D->levels, D->levels + (size_t)d * D->n_comp);
    h->coefs.assign(D->coefs, D->coefs + D->n_comp);
    h->gauss_n.assign(D->gauss_nodes, D->gauss_nodes + h->q);
    h->gauss_w.assign(D->gauss_weights, D->gauss_weights + h->q);
    // geometry
    h->geo = GeoInfo{};
    h->geo.d = d;
    int64_t koff = 0, ncp = 1;
    for (int k = 0; k < d; ++k) {
        int gdeg = D->geo_degree[k], gnk = D->geo_nknots[k];
        if (gdeg < 1 || gdeg >= GEO_PMAX || gnk < 2 * (gdeg + 1)) {
            set_error("geometry knot vector invalid or degree > 7");
            return SGIGA_ERR_VALUE;
        }
        h->geo.deg[k] = gdeg; h->geo.nk[k] = gnk; h->geo.n[k] = gnk - gdeg - 1;
        h->geo.knot_off[k] = koff;
        koff += gnk;
        ncp *= h->geo.n[k];
    }
    h->geo_knots.assign(D->geo_knots, D->geo_knots + koff);
    h->geo_hw.assign(D->geo_hw, D->geo_hw + ncp * (d + 1));
    // knot tables per (axis, level) actually used
    const int L = D->max_level + 1;
    h->tab_of.assign((size_t)d * L, -1);
    h->tabs.clear();
    h->bp_host.clear();
    int64_t knots_tot = 0, vals_tot = 0, qp_tot = 0;
    for (int c = 0; c < D->n_comp; ++c)
        for (int k = 0; k < d; ++k) {
            int lv = D->levels[c * d + k];
            if (lv < 0 || lv > D->max_level) { set_error("level outside [0, max_level]"); return SGIGA_ERR_VALUE; }
            int key = k * L + lv;
            if (h->tab_of[key] >= 0) continue;
            if (D->bp_offset[key] < 0 || D->bp_count[key] < 2) {
                set_error("missing breakpoint table for an (axis, level) pair");
                return SGIGA_ERR_VALUE;
            }
            const double* bp = D->breakpoints + D->bp_offset[key];
            int nbp = D->bp_count[key];
            if (bp[0] != 0.0 || bp[nbp - 1] != 1.0) { set_error("breakpoints must start at 0 and end at 1"); return SGIGA_ERR_VALUE; }
            for (int i = 1; i < nbp; ++i)
                if (!(bp[i] > bp[i - 1])) { set_error("breakpoints must be strictly increasing"); return SGIGA_ERR_VALUE; }
            TabInfo T{};
            T.axis = k; T.level = lv; T.nel = nbp - 1;
            T.nk = 2 * (p + 1) + (T.nel - 1) * h->mu;
            T.n = T.nk - p - 1;
            T.uniform = (T.nel & (T.nel - 1)) == 0;
            for (int i = 0; i < nbp && T.uniform; ++i)
                if (bp[i] != (double)i / (double)T.nel) T.uniform = 0;
            T.bp_off = (int64_t)h->bp_host.size();
            h->bp_host.insert(h->bp_host.end(), bp, bp + nbp);
            T.knot_off = knots_tot;
            knots_tot += T.nk;
            T.val_off = vals_tot;
            vals_tot += 2LL * T.nel * h->q * (p + 1);
            T.qp_off = qp_tot;
            T.geo_off = qp_tot;
            qp_tot += (int64_t)T.nel * h->q;
            h->tab_of[key] = (int)h->tabs.size();
            h->tabs.push_back(T);
        }
    h->total_knots = knots_tot;
    h->total_tabvals = vals_tot;
    h->total_tabqp = qp_tot;

    // components
    h->comps.assign(D->n_comp, CompInfo{});
    h->pencils.clear(); h->blocks2.clear(); h->chunks.clear(); h->small_comps.clear(); h->large_comps.clear(); h->slotoff.clear();
    int64_t vec = 0, mat = 0, qpo = 0, dof = 0, rows_tot = 0, nqp_tot = 0;
    const int W = 2 * p + 1, nG = d * (d + 1) / 2 + 1;
    h->max_slots_comp = 0;
    for (int c = 0; c < D->n_comp; ++c) {
        CompInfo& C = h->comps[c];
        C.coef = D->coefs[c];
        int mmax = -1, s = d - 1;
        for (int k = 0; k < d; ++k) {
            const TabInfo& T = h->tabs[h->tab_of[k * L + D->levels[c * d + k]]];
            C.lv[k] = T.level; C.tab[k] = h->tab_of[k * L + T.level];
            C.n[k] = T.n; C.m[k] = std::max(0, T.n - 2); C.nel[k] = T.nel;
            C.S[k] = C.m[k] <= W ? std::max(1, C.m[k]) : W;
            C.absm[k] = C.m[k] <= W;
        }
        for (int k = d - 1; k >= 0; --k)
            if (C.m[k] > mmax) { mmax = C.m[k]; s = k; }
        // assembly stream axis: the longest by default (line-FD components
        // need their long axis there); small components solved by the FD
        // kernel (every axis <= FD_MMAX functions, <= 2048 rows) stream along
        // their SHORTEST axis instead -- many short pencils rather than a few
        // long ones (the cfg2 makespan was one long pencil), fewer halo planes
        // (the tiled 3-D assembly keeps the longest axis: its tiles cover the
        // thin cross-section, so a long stream axis is what it wants)
        {
            int ls = 0;
            for (int k = 0; k < d; ++k) ls += C.lv[k];
            C.tile3 = tile3_eligible(h) && std::ldexp(1.0, ls) >= TILE3_MIN_ELEMENTS ? 1 : 0;
        }
        if (!C.tile3) {
            int64_t rows_c = 1;
            bool fd_axes = true;
            for (int k = 0; k < d; ++k) { rows_c *= std::max(0, C.m[k]); fd_axes = fd_axes && C.m[k] <= FD_MMAX; }
            if (d >= 2 && fd_axes && rows_c <= 2048 && !(d == 2 && mmax > FD_FULL_MMAX2)) {
                int mmin = 1 << 30;
                for (int k = d - 1; k >= 0; --k)
                    if (C.m[k] < mmin) { mmin = C.m[k]; s = k; }
            }
        }
        int j = 0;
        for (int k = 0; k < d; ++k) if (k != s) C.ax[j++] = k;
        C.ax[d - 1] = s;
        // 3-D: the thinner cross-section axis is a = ax[1] (innermost in the
        // metric storage; the tiled assembly covers it with one union window)
        if (d == 3 && C.m[C.ax[1]] > C.m[C.ax[0]]) std::swap(C.ax[0], C.ax[1]);
        C.rows = 1; C.nslots = 1; C.ndofs = 1; C.nqp = 1;
        for (int k = 0; k < d; ++k) {
            C.rows *= C.m[k]; C.nslots *= C.S[k]; C.ndofs *= C.n[k];
            C.nqp *= (int64_t)C.nel[k] * h->q;
        }
        int64_t pr = 1, ps = 1;
        for (int jj = d - 1; jj >= 0; --jj) {
            int k = C.ax[jj];
            C.rs[k] = pr; pr *= C.m[k];
            C.ss[k] = ps; ps *= C.S[k];
        }
        // qp storage order: stream axis s = ax[d-1] outermost, tile axis
        // a = ax[d-2] innermost (a pencil's plane window is contiguous in a);
        // 2-D components assembled by k_assembly2d: the tile axis (the
        // longer one, walk2d_axis) innermost, so a walk line is contiguous
        int64_t pq = 1;
        const int qorder[3] = {d >= 2 ? C.ax[d - 2] : C.ax[0], d >= 3 ? C.ax[0] : C.ax[d - 1], C.ax[d - 1]};
        const bool asm2d = d == 2 && h->mu == 1 && h->q == p + 1 && !h->opt.generic_assembly;
        for (int jj = 0; jj < d; ++jj) {
            int k = (d == 1) ? C.ax[0]
                             : (d == 2 ? (asm2d ? (jj == 0 ? 1 - walk2d_axis(C) : walk2d_axis(C))
                                                : (jj == 0 ? C.ax[0] : C.ax[1]))
                                       : qorder[jj]);
            C.qs[k] = pq;
            pq *= (int64_t)C.nel[k] * h->q;
        }
        C.halo = 0;
        for (int k = 0; k < d; ++k) if (!C.absm[k]) C.halo += (int64_t)p * C.rs[k];
        // slot offsets in the stencil's linear slot order
        C.so_off = (int64_t)h->slotoff.size();
        for (int64_t t = 0; t < C.nslots; ++t) {
            int64_t off = 0;
            for (int k = 0; k < d; ++k) {
                int sk = (int)((t / C.ss[k]) % C.S[k]);
                off += (int64_t)(C.absm[k] ? sk : sk - p) * C.rs[k];
            }
            h->slotoff.push_back((int)off);
        }
        C.vec_off = vec + C.halo;
        vec += C.rows + 2 * C.halo;
        C.mat_off = mat;
        mat += C.rows * C.nslots;
        C.qp_off = qpo;
        qpo += (int64_t)nG * C.nqp;
        C.dof_off = dof;
        dof += C.ndofs;
        rows_tot += C.rows;
        nqp_tot += C.nqp;
        h->max_slots_comp = std::max<int>(h->max_slots_comp, (int)C.nslots);
        if (C.rows == 0) { C.small = 0; C.nchunks = 0; C.chunk_off = (int64_t)h->chunks.size(); continue; }
        C.small = (C.rows <= 2048 && (6 * C.rows + 2 * C.halo + 64) * 8 <= 200 * 1024) ? 1 : 0;
        (C.small ? h->small_comps : h->large_comps).push_back(c);
        C.chunk_off = (int64_t)h->chunks.size();
        C.nchunks = (int)((C.rows + 255) / 256);
        for (int i = 0; i < C.nchunks; ++i) {
            Chunk ch;
            ch.comp = c; ch.row0 = i * 256; ch.idx = i;
            ch.nrow = (int)std::min<int64_t>(256, C.rows - (int64_t)i * 256);
            h->chunks.push_back(ch);
        }
    }
    // FD-preconditioned CG for the small components whose axes all fit the
    // one-CTA eigen kernel (<= FD_MMAX interior functions) and whose vectors
    // fit shared memory; the others keep the Jacobi-PCG paths
    {
        const bool fd_on = !h->opt.no_fd && !(D->flags & SGIGA_FLAG_ASSEMBLY_ONLY);
        const int ntab = (int)h->tabs.size();
        h->fd_comps.clear(); h->fd_uniq.clear();
        h->fd_uoff.assign(ntab, 0); h->fd_loff.assign(ntab, 0);
        h->fd_u_total = 0; h->fd_l_total = 0;
        std::vector<char> used(ntab, 0);
        std::vector<int> keep_small, keep_large;
        h->fdl_comps.clear();
        h->fdg_comps.clear();
        h->fdl_off.assign(h->comps.size(), -1);
        h->fdl_total = 0;
        for (int c = 0; c < D->n_comp; ++c) {
            CompInfo& C = h->comps[c];
            C.fd = 0;
            if (!C.rows) continue;
            const bool was_small = C.small != 0;
            bool all_ok = fd_on, others_ok = fd_on;
            for (int k = 0; k < d; ++k) {
                const bool ok_k = C.m[k] >= 1 && C.m[k] <= FD_MMAX;
                all_ok = all_ok && ok_k;
                if (k != C.ax[d - 1]) others_ok = others_ok && ok_k;
            }
            if (all_ok && C.rows >= FDG_MIN_ROWS) {   // whole-GPU FD-PCG (cooperative grid)
                C.fd = 3;
                C.small = 1;   // keeps the chunked Jacobi kernels away from it
                h->fdg_comps.push_back(c);
                for (int k = 0; k < d; ++k) used[C.tab[k]] = 1;
            } else if (all_ok && was_small && fd_comp_smem(C, d) <= 200 * 1024 &&
                       !(d == 2 && C.m[C.ax[d - 1]] > FD_FULL_MMAX2)) {   // one CTA, everything in smem
                C.fd = 1;
                h->fd_comps.push_back(c);
                for (int k = 0; k < d; ++k) used[C.tab[k]] = 1;
            } else if (others_ok && C.m[C.ax[d - 1]] >= 1) {   // line FD: banded solves along the stream axis
                C.fd = 2;
                C.small = 1;   // keeps the chunked Jacobi kernels away from it
                h->fdl_comps.push_back(c);
                for (int k = 0; k < d; ++k)
                    if (k != C.ax[d - 1]) used[C.tab[k]] = 1;
                int64_t nl = 1;
                for (int k = 0; k < d; ++k) if (k != C.ax[d - 1]) nl *= C.m[k];
                const int64_t ms = C.m[C.ax[d - 1]];
                h->fdl_off[c] = h->fdl_total;
                h->fdl_total += (2 + nl) * ms * (p + 1);   // K_s, M_s bands + one factor per line
            } else {
                (was_small ? keep_small : keep_large).push_back(c);
            }
        }
        h->small_comps.swap(keep_small);
        h->large_comps.swap(keep_large);
        // line-FD / FD solves are issued longest first (LPT over the waves of
        // clusters / CTAs): the cost of a component ~ its stored stencil
        auto by_cost = [&](int a, int b) {
            const int64_t ca = h->comps[a].rows * h->comps[a].nslots, cb = h->comps[b].rows * h->comps[b].nslots;
            return ca != cb ? ca > cb : a < b;
        };
        std::stable_sort(h->fdl_comps.begin(), h->fdl_comps.end(), by_cost);
        std::stable_sort(h->fd_comps.begin(), h->fd_comps.end(), by_cost);
        // tables with identical knot vectors share one factorisation
        for (int t = 0; t < ntab; ++t) {
            if (!used[t]) continue;
            const TabInfo& T = h->tabs[t];
            int src = -1;
            for (int u : h->fd_uniq) {
                const TabInfo& Tu = h->tabs[u];
                if (Tu.nel == T.nel &&
                    std::equal(h->bp_host.begin() + T.bp_off, h->bp_host.begin() + T.bp_off + T.nel + 1,
                               h->bp_host.begin() + Tu.bp_off)) { src = u; break; }
            }
            if (src >= 0) { h->fd_uoff[t] = h->fd_uoff[src]; h->fd_loff[t] = h->fd_loff[src]; continue; }
            const int64_t m = T.n - 2;
            h->fd_uniq.push_back(t);
            h->fd_uoff[t] = h->fd_u_total; h->fd_u_total += m * m;
            h->fd_loff[t] = h->fd_l_total; h->fd_l_total += m;
        }
    }
    // assembly pencils: tile rows along ax[d-2], ax[d-3]; segments of SEG
    // rows along the stream axis.  A pencil walks its elements one quadrature
    // plane at a time, so its cost is ~ planes (+ a fixed setup); a segment
    // recomputes a p-element halo.  SEG minimises the estimated makespan
    // max(longest pencil, total / resident CTAs); pencils are issued longest
    // first (LPT), so the long ones start in the first wave.
    auto seg_elems = [&](const CompInfo& C, int r0, int r1) {
        const int nel_s = C.nel[C.ax[d - 1]];
        const int ef = std::max(0, r0 - p), el = std::min(r1 - 1, nel_s - 1);
        return std::max(0, el - ef + 1);
    };
    int nsm = 148, dev = 0;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    const double slots = 2.0 * nsm, setup = 2.0;   // 2 resident CTAs/SM; setup in elements
    int SEG = 1 << 20;
    {
        double best = 1e300;
        for (int cand : {1 << 20, 128, 64, 48, 32, 24, 16, 12, 8, 6, 4}) {
            double tot = 0, mx = 0;
            for (const CompInfo& C : h->comps) {
                if (!C.rows) continue;
                const double cross = (double)(d >= 2 ? C.m[C.ax[d - 2]] : 1) * (d >= 3 ? C.m[C.ax[d - 3]] : 1);
                const int ms = C.m[C.ax[d - 1]];
                for (int r0 = 1; r0 < 1 + ms; r0 += cand) {
                    const double cost = seg_elems(C, r0, std::min(1 + ms, r0 + cand)) + setup;
                    tot += cost * cross;
                    mx = std::max(mx, cost);
                }
            }
            const double span = std::max(mx, tot / slots);
            if (span < best * 0.97) { best = span; SEG = cand; }
        }
    }
    for (int c = 0; c < D->n_comp; ++c) {
        const CompInfo& C = h->comps[c];
        if (!C.rows) continue;
        int s = C.ax[d - 1];
        int na = d >= 2 ? C.m[C.ax[d - 2]] : 1, nb = d >= 3 ? C.m[C.ax[d - 3]] : 1;
        int ms = C.m[s];
        int nseg = (ms + SEG - 1) / SEG;
        for (int ib = 0; ib < nb; ++ib)
            for (int ia = 0; ia < na; ++ia)
                for (int sg = 0; sg < nseg; ++sg) {
                    Pencil pc;
                    pc.comp = c;
                    pc.ia = d >= 2 ? ia + 1 : 0;
                    pc.ib = d >= 3 ? ib + 1 : 0;
                    pc.r0 = 1 + sg * SEG;
                    pc.r1 = (int)std::min<int64_t>(1 + ms, 1 + (int64_t)(sg + 1) * SEG);
                    h->pencils.push_back(pc);
                }
    }
    // the pencils of components the tiled kernel does not take come first
    // (launched alone when the tiled kernel runs), each group longest first
    std::stable_sort(h->pencils.begin(), h->pencils.end(), [&](const Pencil& x, const Pencil& y) {
        const int tx = h->comps[x.comp].tile3, ty = h->comps[y.comp].tile3;
        if (tx != ty) return tx < ty;
        return seg_elems(h->comps[x.comp], x.r0, x.r1) > seg_elems(h->comps[y.comp], y.r0, y.r1);
    });
    h->n_pencils_other = 0;
    for (const Pencil& pc : h->pencils) h->n_pencils_other += h->comps[pc.comp].tile3 ? 0 : 1;
    h->asm_seg = SEG;
    // 2-D components (maximal regularity, q = p + 1): blocks of up to ASM2_BA
    // tile rows x a segment of the walk axis for k_assembly2d.  A block walks
    // the SHORTER axis (few barrier intervals of full width -- a thin tile
    // walked along a long axis is a chain of near-empty intervals) and tiles
    // the longer one; the stencil's row order is unaffected.  Cost of a block
    // ~ setup + its walk elements x (tile rows + window halo); the segment
    // length minimises max(longest block, total / resident CTAs)
    if (d == 2 && h->mu == 1 && h->q == p + 1 && !h->opt.generic_assembly) {
        const int BA = ASM2_BA;
        auto walk_of = [&](const CompInfo& C) { return walk2d_axis(C); };
        auto seg_w = [&](const CompInfo& C, int r0, int r1) {
            const int nel_w = C.nel[walk_of(C)];
            const int ef = std::max(0, r0 - p), el = std::min(r1 - 1, nel_w - 1);
            return std::max(0, el - ef + 1);
        };
        auto split_a = [&](const CompInfo& C, std::vector<std::pair<int, int>>& out) {
            const int ma = C.m[1 - walk_of(C)];
            const int nb = (ma + BA - 1) / BA;
            for (int b = 0, start = 0; b < nb; ++b) {
                const int cnt = (ma - start + (nb - b) - 1) / (nb - b);
                out.push_back({1 + start, cnt});
                start += cnt;
            }
        };
        const double slots2 = 2.0 * nsm;
        int SEG2 = 1 << 20;
        double best = 1e300;
        for (int cand : {1 << 20, 64, 32, 16, 8, 4}) {
            double tot = 0, mx = 0;
            for (const CompInfo& C : h->comps) {
                if (!C.rows) continue;
                std::vector<std::pair<int, int>> ab;
                split_a(C, ab);
                const int ms = C.m[walk_of(C)];
                for (auto& [ia0, na] : ab)
                    for (int r0 = 1; r0 < 1 + ms; r0 += cand) {
                        const double cost = (seg_w(C, r0, std::min(1 + ms, r0 + cand)) + 3.0) * (na + p + 2.0);
                        tot += cost;
                        mx = std::max(mx, cost);
                    }
            }
            const double span = std::max(mx, tot / slots2);
            if (span < best * 0.97) { best = span; SEG2 = cand; }
        }
        for (int c = 0; c < D->n_comp; ++c) {
            const CompInfo& C = h->comps[c];
            if (!C.rows) continue;
            std::vector<std::pair<int, int>> ab;
            split_a(C, ab);
            const int ms = C.m[walk_of(C)];
            for (auto& [ia0, na] : ab)
                for (int r0 = 1; r0 < 1 + ms; r0 += SEG2) {
                    Block2 bk;
                    bk.comp = c; bk.walk = walk_of(C); bk.ia0 = ia0; bk.na = na;
                    bk.r0 = r0; bk.r1 = std::min(1 + ms, r0 + SEG2);
                    h->blocks2.push_back(bk);
                }
        }
        std::stable_sort(h->blocks2.begin(), h->blocks2.end(), [&](const Block2& x, const Block2& y) {
            return seg_w(h->comps[x.comp], x.r0, x.r1) * (x.na + p) > seg_w(h->comps[y.comp], y.r0, y.r1) * (y.na + p);
        });
    }
    h->total_vec = vec; h->total_slots = mat; h->total_qp = nqp_tot; h->total_rows = rows_tot;
    {   // k_metric: component of each 256-point CTA's first point
        h->mcomp.assign((size_t)((nqp_tot + 255) / 256), 0);
        int c = 0;
        int64_t end = h->comps.empty() ? 0 : h->comps[0].nqp;
        for (size_t b = 0; b < h->mcomp.size(); ++b) {
            const int64_t g0 = (int64_t)b * 256;
            while (c + 1 < (int)h->comps.size() && g0 >= end) end += h->comps[++c].nqp;
            h->mcomp[b] = c;
        }
    }
    h->total_dofs = dof;
    if (assembly_smem_bytes(h) > 227 * 1024) {
        set_error("quadrature/degree combination exceeds the assembly kernel's shared memory");
        return SGIGA_ERR_VALUE;
    }
    return SGIGA_OK;
}

static int upload_all(Handle* h) {
    cudaStream_t s = h->stream;
    h->tmaps_state = 0;   // tensor maps follow the component table
    h->tiles3_state = 0;
    free_box(h);
    h->stencil_zeroed = false;
    h->metric_offdiag_zeroed = false;
    if (!h->mcomp.empty())
        SG_CUDA(cudaMemcpyAsync(h->d_mcomp, h->mcomp.data(), sizeof(int) * h->mcomp.size(), cudaMemcpyHostToDevice, s));
    SG_CUDA(cudaMemcpyAsync(h->d_comps, h->comps.data(), sizeof(CompInfo) * h->comps.size(), cudaMemcpyHostToDevice, s));
    SG_CUDA(cudaMemcpyAsync(h->d_tabs, h->tabs.data(), sizeof(TabInfo) * h->tabs.size(), cudaMemcpyHostToDevice, s));
    SG_CUDA(cudaMemcpyAsync(h->d_geo, &h->geo, sizeof(GeoInfo), cudaMemcpyHostToDevice, s));
    if (!h->pencils.empty())
        SG_CUDA(cudaMemcpyAsync(h->d_pencils, h->pencils.data(), sizeof(Pencil) * h->pencils.size(), cudaMemcpyHostToDevice, s));
    if (!h->blocks2.empty())
        SG_CUDA(cudaMemcpyAsync(h->d_blocks2, h->blocks2.data(), sizeof(Block2) * h->blocks2.size(), cudaMemcpyHostToDevice, s));
    if (!h->chunks.empty())
        SG_CUDA(cudaMemcpyAsync(h->d_chunks, h->chunks.data(), sizeof(Chunk) * h->chunks.size(), cudaMemcpyHostToDevice, s));
    if (!h->small_comps.empty())
        SG_CUDA(cudaMemcpyAsync(h->d_small, h->small_comps.data(), sizeof(int) * h->small_comps.size(), cudaMemcpyHostToDevice, s));
    if (!h->slotoff.empty())
        SG_CUDA(cudaMemcpyAsync(h->d_slotoff, h->slotoff.data(), sizeof(int) * h->slotoff.size(), cudaMemcpyHostToDevice, s));
    if (!h->fdg_comps.empty())
        SG_CUDA(cudaMemcpyAsync(h->d_fdg_list, h->fdg_comps.data(), sizeof(int) * h->fdg_comps.size(), cudaMemcpyHostToDevice, s));
    if (!h->fdl_comps.empty()) {
        SG_CUDA(cudaMemcpyAsync(h->d_fdl_list, h->fdl_comps.data(), sizeof(int) * h->fdl_comps.size(), cudaMemcpyHostToDevice, s));
        SG_CUDA(cudaMemcpyAsync(h->d_fdl_off, h->fdl_off.data(), sizeof(int64_t) * h->fdl_off.size(), cudaMemcpyHostToDevice, s));
    }
    if (!h->fd_uniq.empty()) {
        SG_CUDA(cudaMemcpyAsync(h->d_fd_uniq, h->fd_uniq.data(), sizeof(int) * h->fd_uniq.size(), cudaMemcpyHostToDevice, s));
        SG_CUDA(cudaMemcpyAsync(h->d_fd_uoff, h->fd_uoff.data(), sizeof(int64_t) * h->fd_uoff.size(), cudaMemcpyHostToDevice, s));
        SG_CUDA(cudaMemcpyAsync(h->d_fd_loff, h->fd_loff.data(), sizeof(int64_t) * h->fd_loff.size(), cudaMemcpyHostToDevice, s));
    }
    if (!h->fd_comps.empty())
        SG_CUDA(cudaMemcpyAsync(h->d_fdlist, h->fd_comps.data(), sizeof(int) * h->fd_comps.size(), cudaMemcpyHostToDevice, s));
    SG_CUDA(cudaMemcpyAsync(h->d_bp, h->bp_host.data(), sizeof(double) * h->bp_host.size(), cudaMemcpyHostToDevice, s));
    {   // open knot vectors: exact metadata of the breakpoints (make_open_knot_vector,
        // splines.py:83-110 -- [0]*(p+1), interior breakpoints with multiplicity mu,
        // [1]*(p+1)), uploaded with the descriptor
        h->knots_host.assign((size_t)h->total_knots, 0.0);
        for (const TabInfo& T : h->tabs) {
            const double* b = h->bp_host.data() + T.bp_off;
            const int nk = 2 * (h->p + 1) + (T.nel - 1) * h->mu;
            for (int pos = 0; pos < nk; ++pos)
                h->knots_host[T.knot_off + pos] =
                    pos <= h->p ? 0.0 : (pos >= nk - (h->p + 1) ? 1.0 : b[1 + (pos - (h->p + 1)) / h->mu]);
        }
        if (!h->knots_host.empty())
            SG_CUDA(cudaMemcpyAsync(h->d_knots, h->knots_host.data(), sizeof(double) * h->knots_host.size(),
                                    cudaMemcpyHostToDevice, s));
    }
    SG_CUDA(cudaMemcpyAsync(h->d_geo_knots, h->geo_knots.data(), sizeof(double) * h->geo_knots.size(), cudaMemcpyHostToDevice, s));
    SG_CUDA(cudaMemcpyAsync(h->d_geo_hw, h->geo_hw.data(), sizeof(double) * h->geo_hw.size(), cudaMemcpyHostToDevice, s));
    // gauss + cumulative index tables
    std::vector<char> blob;
    std::vector<double> g(2 * h->q);
    for (int i = 0; i < h->q; ++i) { g[i] = h->gauss_n[i]; g[h->q + i] = h->gauss_w[i]; }
    std::vector<int64_t> cum;
    int64_t acc = 0;
    cum.push_back(0);
    for (auto& T : h->tabs) { acc += (int64_t)T.nel * h->q; cum.push_back(acc); }
    acc = 0;
    cum.push_back(0);
    for (auto& C : h->comps) { acc += C.nqp; cum.push_back(acc); }
    acc = 0;
    cum.push_back(0);
    for (auto& C : h->comps) { acc += C.ndofs; cum.push_back(acc); }
    blob.resize(g.size() * 8 + cum.size() * 8);
    memcpy(blob.data(), g.data(), g.size() * 8);
    memcpy(blob.data() + g.size() * 8, cum.data(), cum.size() * 8);
    SG_CUDA(cudaMemcpyAsync(h->d_gauss, blob.data(), blob.size(), cudaMemcpyHostToDevice, s));
    SG_CUDA(cudaStreamSynchronize(s));  // blob is a host temporary
    h->tables_ready = false;
    h->assembled = false;
    h->solved = false;
    return SGIGA_OK;
}

// device error flags: the copy is enqueued on the stream, decoded after the
// caller's (single) synchronisation
static int decode_err(Handle* h);
static int check_err(Handle* h) {
    SG_CUDA(cudaMemcpyAsync(h->h_err, h->d_err, sizeof(int), cudaMemcpyDeviceToHost, h->stream));
    SG_CUDA(cudaStreamSynchronize(h->stream));
    return decode_err(h);
}
static int decode_err(Handle* h) {
    const int e = *h->h_err;
    *h->h_err = 0;
    if (e & ERRF_GEOMETRY) {
        set_error("geometry map is degenerate: det J <= 0 at a quadrature point");
        SG_CUDA(cudaMemsetAsync(h->d_err, 0, sizeof(int), h->stream));
        return SGIGA_ERR_GEOMETRY;
    }
    if (e & 8) {
        set_error("small-path PCG: thread-block cluster launched with an unexpected shape");
        SG_CUDA(cudaMemsetAsync(h->d_err, 0, sizeof(int), h->stream));
        return SGIGA_ERR_CUDA;
    }
    if (e & ERRF_POINTS) {
        set_error("evaluation points must lie in [0, 1]^d");
        SG_CUDA(cudaMemsetAsync(h->d_err, 0, sizeof(int), h->stream));
        return SGIGA_ERR_VALUE;
    }
    if (e & ERRF_SPAN) {
        set_error("quadrature node escaped its element");
        SG_CUDA(cudaMemsetAsync(h->d_err, 0, sizeof(int), h->stream));
        return SGIGA_ERR_VALUE;
    }
    return SGIGA_OK;
}

static int ensure_tables(Handle* h) {
    if (h->tables_ready) return SGIGA_OK;
    h->kstart(0);
    SG_CUDA(launch_basis_tables(h));   // (the knot vectors are uploaded with the descriptor)
    h->kstop(0);
    h->tables_ready = true;
    return SGIGA_OK;
}

}  // namespace sgiga

using namespace sgiga;

extern "C" {

const char* sgiga_last_error(void) { return g_last_error.c_str(); }

int sgiga_device_count(int32_t* n) {
    int c = 0;
    cudaError_t e = cudaGetDeviceCount(&c);
    if (e != cudaSuccess) { *n = 0; set_error(cudaGetErrorString(e)); return SGIGA_ERR_CUDA; }
    *n = c;
    return SGIGA_OK;
}

int sgiga_create(const sgiga_problem_desc* desc, void* stream, sgiga_handle** out) {
    if (!desc || !out) { set_error("null argument"); return SGIGA_ERR_VALUE; }
    *out = nullptr;
    Handle* h = new Handle();
    int st = build_tables(h, desc);
    if (st) { delete h; return st; }
    cudaError_t e = cudaGetDevice(&h->dev);
    if (e != cudaSuccess) { set_error(std::string("no CUDA device: ") + cudaGetErrorString(e)); delete h; return SGIGA_ERR_CUDA; }
    if (stream) {
        h->stream = (cudaStream_t)stream;
    } else {
        e = cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking);
        if (e != cudaSuccess) { set_error(cudaGetErrorString(e)); delete h; return SGIGA_ERR_CUDA; }
        h->own_stream = true;
    }
    const int nG = h->nG();
    cudaError_t ea = cudaSuccess;
#define A_(ptr, n) if (ea == cudaSuccess) ea = dalloc(&h->ptr, (size_t)(n))
    A_(d_comps, h->comps.size());
    A_(d_tabs, h->tabs.size());
    A_(d_geo, 1);
    A_(d_pencils, h->pencils.size());
    A_(d_blocks2, h->blocks2.size());
    A_(d_chunks, h->chunks.size());
    A_(d_small, h->small_comps.size());
    A_(d_large, h->large_comps.size());
    A_(d_bp, h->bp_host.size());
    A_(d_knots, h->total_knots);
    A_(d_gauss, 2 * h->q + (h->tabs.size() + 1) + 2 * (h->ncomp + 1));
    A_(d_tabvals, h->total_tabvals);
    A_(d_qx, h->total_tabqp);
    A_(d_qw, h->total_tabqp);
    A_(d_geob, h->total_tabqp * 2 * GEO_PMAX);
    A_(d_geofirst, h->total_tabqp);
    A_(d_geo_knots, h->geo_knots.size());
    A_(d_geo_hw, h->geo_hw.size());
    A_(d_G, nG * h->total_qp);
    A_(d_stencil, h->total_slots);
    A_(d_rhs, h->total_vec);
    A_(d_dinv, h->total_vec);
    A_(d_x, h->total_vec);
    A_(d_r, h->total_vec);
    A_(d_z, h->total_vec);
    A_(d_p, h->total_vec);
    A_(d_q, h->total_vec);
    A_(d_q2, h->total_vec);
    A_(d_coef, h->total_dofs + 2);   // +2: the combine's 16-byte row loads may read past the end
    A_(d_cg, h->ncomp);
    A_(d_part, 3 * h->chunks.size());
    A_(d_err, 1);
    A_(d_active_count, 4);        // [active comps, active chunks, host copy of chunks]
    A_(d_alist, h->chunks.size());
    A_(d_relres, h->ncomp);
    A_(d_slotoff, h->slotoff.size());
    A_(d_chist, COMBINE_SORT_BINS);
    A_(d_fdlist, h->fd_comps.size());
    A_(d_fd_uniq, h->fd_uniq.size());
    A_(d_fd_uoff, h->tabs.size());
    A_(d_fd_loff, h->tabs.size());
    A_(d_fdU, h->fd_u_total);
    A_(d_fdL, h->fd_l_total);
    A_(d_fdl_list, h->fdl_comps.size());
    A_(d_fdg_list, h->fdg_comps.size());
    A_(d_fdg_part, 2 * FDG_MAX_CTAS);
    A_(d_fdg_ckpart, h->fdg_comps.size() * MAXD * 256);   // k_fd_metric_scale_part chunk partials
    A_(d_fdl_off, h->comps.size());
    A_(d_fdl, h->fdl_total);
    A_(d_ck, (int64_t)MAXD * h->ncomp);
    A_(d_mcomp, h->mcomp.size());
    if (ea == cudaSuccess && !h->d_ticket) {
        ea = cudaMalloc(&h->d_ticket, sizeof(unsigned));
        if (ea == cudaSuccess) ea = cudaMemset(h->d_ticket, 0, sizeof(unsigned));
    }
#undef A_
    // side streams at the highest priority: their few CTAs (FD set-up, point
    // sort) are scheduled as soon as an SM frees up instead of queueing behind
    // the thousands of assembly CTAs launched before them
    int prio_lo = 0, prio_hi = 0;
    if (ea == cudaSuccess) ea = cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi);
    if (ea == cudaSuccess) ea = cudaStreamCreateWithPriority(&h->stream2, cudaStreamNonBlocking, prio_hi);
    if (ea == cudaSuccess) ea = cudaEventCreateWithFlags(&h->fd_fork, cudaEventDisableTiming);
    if (ea == cudaSuccess) ea = cudaEventCreateWithFlags(&h->fd_join, cudaEventDisableTiming);
    if (ea == cudaSuccess) ea = cudaEventCreateWithFlags(&h->fd_metric, cudaEventDisableTiming);
    if (ea == cudaSuccess) ea = cudaEventCreateWithFlags(&h->pcg_fork, cudaEventDisableTiming);
    if (ea == cudaSuccess) ea = cudaEventCreateWithFlags(&h->pcg_join, cudaEventDisableTiming);
    if (ea == cudaSuccess) ea = cudaStreamCreateWithPriority(&h->stream3, cudaStreamNonBlocking, prio_hi);
    if (ea == cudaSuccess) ea = cudaEventCreateWithFlags(&h->cs_fork, cudaEventDisableTiming);
    if (ea == cudaSuccess) ea = cudaEventCreateWithFlags(&h->cs_join, cudaEventDisableTiming);
    if (ea == cudaSuccess) ea = cudaMallocHost(reinterpret_cast<void**>(&h->h_pinned_flag), sizeof(int) * 4);
    // mapped pinned mirrors: the status kernel writes them directly (no copy nodes)
    if (ea == cudaSuccess) ea = cudaHostAlloc(reinterpret_cast<void**>(&h->h_err), sizeof(int), cudaHostAllocMapped);
    if (ea == cudaSuccess)
        ea = cudaHostAlloc(reinterpret_cast<void**>(&h->h_cg), sizeof(CgState) * std::max(1, h->ncomp), cudaHostAllocMapped);
    if (ea == cudaSuccess)
        ea = cudaHostAlloc(reinterpret_cast<void**>(&h->h_rel), sizeof(double) * std::max(1, h->ncomp), cudaHostAllocMapped);
    if (ea == cudaSuccess) ea = cudaHostAlloc(reinterpret_cast<void**>(&h->h_sticky), sizeof(int), cudaHostAllocMapped);
    if (ea == cudaSuccess) { *h->h_sticky = 0; ea = cudaHostGetDevicePointer(reinterpret_cast<void**>(&h->dh_sticky), h->h_sticky, 0); }
    if (ea == cudaSuccess) ea = cudaHostGetDevicePointer(reinterpret_cast<void**>(&h->dh_err), h->h_err, 0);
    if (ea == cudaSuccess) ea = cudaHostGetDevicePointer(reinterpret_cast<void**>(&h->dh_cg), h->h_cg, 0);
    if (ea == cudaSuccess) ea = cudaHostGetDevicePointer(reinterpret_cast<void**>(&h->dh_rel), h->h_rel, 0);
    if (ea == cudaSuccess) ea = cudaMemsetAsync(h->d_chist, 0, sizeof(int) * COMBINE_SORT_BINS, h->stream);
    for (auto& ev : h->evp)
        if (ea == cudaSuccess) ea = cudaEventCreate(&ev);
    if (ea != cudaSuccess) {
        set_error(std::string("device allocation failed: ") + cudaGetErrorString(ea));
        free_all(h);
        delete h;
        return SGIGA_ERR_CUDA;
    }
    // zero everything that is gathered through halos or reduced
    cudaStream_t s = h->stream;
    double* vecs[] = {h->d_rhs, h->d_dinv, h->d_x, h->d_r, h->d_z, h->d_p, h->d_q, h->d_q2};
    for (double* v : vecs) cudaMemsetAsync(v, 0, sizeof(double) * std::max<int64_t>(1, h->total_vec), s);
    cudaMemsetAsync(h->d_cg, 0, sizeof(CgState) * h->ncomp, s);
    cudaMemsetAsync(h->d_err, 0, sizeof(int), s);
    cudaMemsetAsync(h->d_coef, 0, sizeof(double) * std::max<int64_t>(1, h->total_dofs), s);
    st = upload_all(h);
    if (st) { free_all(h); delete h; return st; }
    h->iters.assign(h->ncomp, 0);
    h->force_generic_assembly = h->opt.generic_assembly;
    h->ktimes = !h->opt.no_ktimes;
    *out = reinterpret_cast<sgiga_handle*>(h);
    return SGIGA_OK;
}

int sgiga_upload(sgiga_handle* hh, const sgiga_problem_desc* desc) {
    Handle* h = reinterpret_cast<Handle*>(hh);
    if (!h || !desc) { set_error("null argument"); return SGIGA_ERR_VALUE; }
    // same-shape re-upload: rebuild the tables on a scratch handle and compare sizes
    Handle tmp;
    int st = build_tables(&tmp, desc);
    if (st) return st;
    if (tmp.total_slots != h->total_slots || tmp.total_qp != h->total_qp ||
        tmp.ncomp != h->ncomp || tmp.tabs.size() != h->tabs.size() || tmp.d != h->d ||
        tmp.p != h->p || tmp.q != h->q || tmp.pencils.size() != h->pencils.size() ||
        tmp.blocks2.size() != h->blocks2.size() ||
        tmp.chunks.size() != h->chunks.size() || tmp.small_comps.size() != h->small_comps.size() ||
        tmp.large_comps.size() != h->large_comps.size() || tmp.slotoff.size() != h->slotoff.size() ||
        tmp.fd_comps.size() != h->fd_comps.size() || tmp.fd_uniq.size() != h->fd_uniq.size() ||
        tmp.fd_u_total != h->fd_u_total || tmp.fd_l_total != h->fd_l_total ||
        tmp.fdl_comps.size() != h->fdl_comps.size() || tmp.fdl_total != h->fdl_total ||
        tmp.fdg_comps.size() != h->fdg_comps.size()) {
        set_error("sgiga_upload: descriptor shape differs from the handle's");
        return SGIGA_ERR_VALUE;
    }
    // an identical descriptor keeps the captured whole-run graph
    auto same_bytes = [](const auto& a, const auto& b) {
        return a.size() == b.size() && (a.empty() || !memcmp(a.data(), b.data(), sizeof(a[0]) * a.size()));
    };
    const bool identical = same_bytes(tmp.levels, h->levels) && same_bytes(tmp.coefs, h->coefs) &&
                           same_bytes(tmp.gauss_n, h->gauss_n) && same_bytes(tmp.gauss_w, h->gauss_w) &&
                           !memcmp(&tmp.geo, &h->geo, sizeof(GeoInfo)) && same_bytes(tmp.geo_knots, h->geo_knots) &&
                           same_bytes(tmp.geo_hw, h->geo_hw) && same_bytes(tmp.bp_host, h->bp_host) &&
                           same_bytes(tmp.comps, h->comps) && same_bytes(tmp.tabs, h->tabs) &&
                           same_bytes(tmp.slotoff, h->slotoff) && same_bytes(tmp.pencils, h->pencils) &&
                           same_bytes(tmp.blocks2, h->blocks2) &&
                           same_bytes(tmp.chunks, h->chunks) && same_bytes(tmp.small_comps, h->small_comps) &&
                           same_bytes(tmp.large_comps, h->large_comps) && same_bytes(tmp.fd_comps, h->fd_comps) &&
                           same_bytes(tmp.fd_uniq, h->fd_uniq) && same_bytes(tmp.fd_uoff, h->fd_uoff) &&
                           same_bytes(tmp.fdl_comps, h->fdl_comps) && same_bytes(tmp.fdl_off, h->fdl_off) &&
                           same_bytes(tmp.fdg_comps, h->fdg_comps) &&
                           tmp.forcing_id == h->forcing_id;
    if (!identical) h->drop_run_graph();
    h->levels.swap(tmp.levels); h->coefs.swap(tmp.coefs);
    h->gauss_n.swap(tmp.gauss_n); h->gauss_w.swap(tmp.gauss_w);
    h->geo = tmp.geo; h->geo_knots.swap(tmp.geo_knots); h->geo_hw.swap(tmp.geo_hw);
    h->bp_host.swap(tmp.bp_host); h->comps.swap(tmp.comps); h->tabs.swap(tmp.tabs);
    h->slotoff.swap(tmp.slotoff);
    h->pencils.swap(tmp.pencils); h->blocks2.swap(tmp.blocks2); h->chunks.swap(tmp.chunks); h->mcomp.swap(tmp.mcomp);
    h->small_comps.swap(tmp.small_comps); h->large_comps.swap(tmp.large_comps);
    h->fd_comps.swap(tmp.fd_comps); h->fd_uniq.swap(tmp.fd_uniq);
    h->fd_uoff.swap(tmp.fd_uoff); h->fd_loff.swap(tmp.fd_loff);
    h->fdl_comps.swap(tmp.fdl_comps); h->fdl_off.swap(tmp.fdl_off); h->fdg_comps.swap(tmp.fdg_comps);
    h->forcing_id = tmp.forcing_id;
    if (identical) return SGIGA_OK;   // device copies are already these bytes
    return upload_all(h);
}

int sgiga_batch_sizes(sgiga_handle* hh, int64_t* total_qp, int64_t* total_rows,
                      int64_t* total_dofs, int64_t* total_slots) {
    Handle* h = reinterpret_cast<Handle*>(hh);
    if (!h) return SGIGA_ERR_VALUE;
    if (total_qp) *total_qp = h->total_qp;
    if (total_rows) *total_rows = h->total_rows;
    if (total_dofs) *total_dofs = h->total_dofs;
    if (total_slots) *total_slots = h->total_slots;
    return SGIGA_OK;
}

int sgiga_component_info(sgiga_handle* hh, int32_t* dims, int64_t* dof_offsets) {
    Handle* h = reinterpret_cast<Handle*>(hh);
    if (!h) return SGIGA_ERR_VALUE;
    for (int c = 0; c < h->ncomp; ++c) {
        if (dims) for (int k = 0; k < h->d; ++k) dims[c * h->d + k] = h->comps[c].n[k];
        if (dof_offsets) dof_offsets[c] = h->comps[c].dof_off;
    }
    if (dof_offsets) dof_offsets[h->ncomp] = h->total_dofs;
    return SGIGA_OK;
}

int sgiga_quad_points_physical(sgiga_handle* hh, double* x_out) {
    Handle* h = reinterpret_cast<Handle*>(hh);
    if (!h || !x_out) return SGIGA_ERR_VALUE;
    if (h->forcing_id != SGIGA_FORCING_HOST) { set_error("only for SGIGA_FORCING_HOST"); return SGIGA_ERR_STATE; }
    if (!h->d_xphys) SG_CUDA(dalloc(&h->d_xphys, h->total_qp * h->d));
    if (!h->d_hostf) {
        SG_CUDA(dalloc(&h->d_hostf, h->total_qp));
        SG_CUDA(cudaMemsetAsync(h->d_hostf, 0, sizeof(double) * std::max<int64_t>(1, h->total_qp), h->stream));
    }
    h->begin_call();
    int st = ensure_tables(h);
    if (st) return st;
    SG_CUDA(launch_metric(h));
    st = check_err(h);
    if (st) return st;
    SG_CUDA(cudaMemcpy(x_out, h->d_xphys, sizeof(double) * h->total_qp * h->d, cudaMemcpyDeviceToHost));
    return SGIGA_OK;
}

int sgiga_set_forcing_density(sgiga_handle* hh, const double* f) {
    Handle* h = reinterpret_cast<Handle*>(hh);
    if (!h || !f) return SGIGA_ERR_VALUE;
    if (!h->d_hostf) SG_CUDA(dalloc(&h->d_hostf, h->total_qp));
    SG_CUDA(cudaMemcpyAsync(h->d_hostf, f, sizeof(double) * h->total_qp, cudaMemcpyHostToDevice, h->stream));
    SG_CUDA(cudaStreamSynchronize(h->stream));
    h->density_ready = true;
    return SGIGA_OK;
}

// ---- the three phases, split into an enqueue part (async, on the
// handle's stream) and a finish part (after one synchronisation) -----------
static int assemble_enqueue(Handle* h) {
    if (h->forcing_id == SGIGA_FORCING_HOST && !h->density_ready) {
        set_error("host forcing: call sgiga_set_forcing_density first");
        return SGIGA_ERR_STATE;
    }
    h->launches[0] = 0;
    h->begin_call();           // assembly always opens a call's launch sequence
    h->pmark(0);
    h->tables_ready = false;   // kernel 1 is part of every assembly pass
    int st = ensure_tables(h);
    if (st) return st;
    if (!h->fd_uniq.empty() || !h->fd_comps.empty() || !h->fdl_comps.empty() || !h->fdg_comps.empty()) {   // FD eigen-factors on the side stream, overlapping the assembly
        SG_CUDA(cudaEventRecord(h->fd_fork, h->stream));
        SG_CUDA(cudaStreamWaitEvent(h->stream2, h->fd_fork, 0));
        SG_CUDA(launch_solve_prologue(h, h->stream2));   // solver state zeroed off the main stream
        SG_CUDA(launch_fd_eigen(h, h->stream2));
        h->fd_pending = true;
    }
    // Kronecker box assembly: c_k is a closed form and the line factors need
    // only kernel 1's tables -- the whole FD set-up runs beside the metric
    const bool fd_early = h->fd_pending && box_assembly_ready(h);
    if (fd_early) {
        SG_CUDA(launch_fd_setup(h, h->stream2));
        SG_CUDA(cudaEventRecord(h->fd_join, h->stream2));
    }
    h->kstart(1);
    SG_CUDA(launch_metric(h));
    h->kstop(1);
    if (h->fd_pending && !fd_early) {   // c_k and the line factors need the metric: side stream again
        SG_CUDA(cudaEventRecord(h->fd_metric, h->stream));
        SG_CUDA(cudaStreamWaitEvent(h->stream2, h->fd_metric, 0));
        SG_CUDA(launch_fd_setup(h, h->stream2));
        SG_CUDA(cudaEventRecord(h->fd_join, h->stream2));
    }
    h->kstart(2);
    SG_CUDA(launch_assembly(h));
    h->kstop(2);
    h->pmark(1);
    return SGIGA_OK;
}

static int solve_enqueue(Handle* h, double rtol, int32_t maxit) {
    if (!(rtol > 0.0)) { set_error("rtol must be positive"); return SGIGA_ERR_VALUE; }
    if (maxit < 1) maxit = 1000000;
    h->launches[1] = 0;
    h->pmark(2);
    // zero the solver state and the active counts (already done on the FD
    // side stream when the assembly forked it: joined before the solve)
    if (!h->fd_pending) SG_CUDA(launch_solve_prologue(h, h->stream));
    int st = run_pcg(h, rtol, maxit);
    if (st) return st;
    h->kstart(5);
    SG_CUDA(launch_residual_check(h));
    SG_CUDA(launch_expand(h));
    h->kstop(5);
    h->pmark(3);
    return SGIGA_OK;
}

// per-component convergence verdict (linsolve.py:49-53 acceptance)
static int solve_finish(Handle* h, int32_t* iters_out, double* relres_out) {
    SG_CUDA(h->elapsed(&h->ms[1], Handle::PHASE_EV + 2, Handle::PHASE_EV + 3));
    h->have_coefs = true;
    h->solved = true;
    int status = SGIGA_OK;
    char buf[256];
    for (int c = 0; c < h->ncomp; ++c) {
        const CompInfo& C = h->comps[c];
        const CgState& cg = h->h_cg[c];
        const double rel = h->h_rel[c];
        h->iters[c] = C.rows ? cg.it : 0;
        if (iters_out) iters_out[c] = h->iters[c];
        if (relres_out) relres_out[c] = C.rows ? rel : 0.0;
        if (!C.rows || cg.bb == 0.0) continue;
        if (!std::isfinite(rel)) {
            snprintf(buf, sizeof buf, "component %d: solve produced non-finite values", c);
            set_error(buf);
            status = SGIGA_ERR_SOLVE;
        } else if (!cg.conv) {
            snprintf(buf, sizeof buf, "component %d: PCG did not converge in %d iterations", c, cg.it);
            set_error(buf);
            status = SGIGA_ERR_SOLVE;
        } else if (rel > 1e-10) {   // linsolve.py:49-53
            snprintf(buf, sizeof buf, "component %d: relative residual %.3e exceeds tol 1.0e-10", c, rel);
            set_error(buf);
            status = SGIGA_ERR_SOLVE;
        }
    }
    return status;
}

// per-handle staging buffers (allocated on the handle's device).  A buffer
// that grows while passes of this handle are still in flight is freed only
// after the handle's streams drain.
static int ensure_scratch(Handle* h, double** buf, size_t* cap, size_t n) {
    if (*cap >= n && *buf) return SGIGA_OK;
    if (*buf) {
        SG_CUDA(cudaStreamSynchronize(h->stream));
        SG_CUDA(cudaStreamSynchronize(h->stream3));
        cudaFree(*buf);
    }
    *buf = nullptr;
    *cap = 0;
    SG_CUDA(cudaMalloc(reinterpret_cast<void**>(buf), std::max<size_t>(n, 1) * sizeof(double)));
    *cap = n;
    return SGIGA_OK;
}

// host points -> device scratch (device = 0 / -1 of sgiga_combine_points)
static int stage_points(Handle* h, const double* pts, int64_t npts, size_t nout, const double** dp,
                        double** dout) {
    int st;
    if ((st = ensure_scratch(h, &h->d_spts, &h->spts_cap, (size_t)npts * h->d))) return st;
    if ((st = ensure_scratch(h, &h->d_sout, &h->sout_cap, nout))) return st;
    SG_CUDA(cudaMemcpyAsync(h->d_spts, pts, sizeof(double) * npts * h->d, cudaMemcpyHostToDevice, h->stream));
    *dp = h->d_spts;
    *dout = h->d_sout;
    return SGIGA_OK;
}

// device points -> device values
static int combine_enqueue(Handle* h, const double* dp, int64_t npts, double* dout, int per_comp,
                           bool* status_fused = nullptr) {
    h->launches[2] = 0;
    h->pmark(4);
    if (h->cs_pending) {   // the point sort ran on the side stream
        SG_CUDA(cudaStreamWaitEvent(h->stream, h->cs_join, 0));
        h->cs_pending = false;
    }
    h->kstart(6);
    SG_CUDA(launch_combine_points(h, dp, npts, dout, per_comp, status_fused));
    h->kstop(6);
    h->pmark(5);
    return SGIGA_OK;
}

int sgiga_assemble(sgiga_handle* hh) {
    Handle* h = reinterpret_cast<Handle*>(hh);
    if (!h) return SGIGA_ERR_VALUE;
    int st = assemble_enqueue(h);
    if (st) return st;
    st = check_err(h);
    if (st) return st;
    SG_CUDA(h->elapsed(&h->ms[0], Handle::PHASE_EV + 0, Handle::PHASE_EV + 1));
    h->assembled = true;
    h->solved = false;
    return SGIGA_OK;
}

int sgiga_solve(sgiga_handle* hh, double rtol, int32_t maxit, int32_t* iters_out,
                double* relres_out) {
    Handle* h = reinterpret_cast<Handle*>(hh);
    if (!h) return SGIGA_ERR_VALUE;
    if (!h->assembled) { set_error("sgiga_solve before sgiga_assemble"); return SGIGA_ERR_STATE; }
    h->begin_call();
    int st = solve_enqueue(h, rtol, maxit);
    if (st) return st;
    SG_CUDA(launch_status(h));
    SG_CUDA(cudaStreamSynchronize(h->stream));   // h_cg / h_rel / h_err are valid after it
    *h->h_sticky = 0;                            // this call's verdict is solve_finish's
    if ((st = decode_err(h))) return st;
    return solve_finish(h, iters_out, relres_out);
}

// Whole-pass CUDA graphs are opt-in (SGIGA_RUN_GRAPH=1): measured on the B200,
// passes enqueued back to back hide the host launch cost anyway (cfg2 0.248
// ms/pass direct vs 0.251 replayed), and in a replayed graph the side-stream
// FD set-up did not overlap the assembly (cfg5 +1 ms)
static bool run_graphs_enabled(const Handle* h) {
    return h->opt.run_graph && !h->opt.pcg_profile && !h->opt.asm_profile && !h->opt.pcg_trace;
}

// enqueue of one whole pass (device pointers): direct launches, capture, or
// replay of the pass graph; no synchronisation
static int run_enqueue(Handle* h, double rtol, int32_t maxit, const double* dp, int64_t npts, double* dout,
                       const double* hsrc = nullptr, int per_comp = 0) {
    int st;
    if (!(rtol > 0.0)) { set_error("rtol must be positive"); return SGIGA_ERR_VALUE; }   // before any launch
    auto enqueue_all = [&]() -> int {
        // the combine's point sort depends on the points only: side stream,
        // overlapping assembly and solve
        h->cs_ready = h->cs_pending = false;
        if (npts > 0) {
            bool sorted = false;
            SG_CUDA(cudaEventRecord(h->cs_fork, h->stream));
            SG_CUDA(cudaStreamWaitEvent(h->stream3, h->cs_fork, 0));
            if (hsrc)   // pinned host points: their upload overlaps assembly and solve too
                SG_CUDA(cudaMemcpyAsync(const_cast<double*>(dp), hsrc, sizeof(double) * npts * h->d,
                                        cudaMemcpyHostToDevice, h->stream3));
            SG_CUDA(launch_combine_sort(h, dp, npts, h->stream3, &sorted));
            SG_CUDA(cudaEventRecord(h->cs_join, h->stream3));
            h->cs_pending = true;
            h->cs_ready = sorted;
        }
        int s2 = assemble_enqueue(h);
        if (!s2) s2 = solve_enqueue(h, rtol, maxit);
        bool fused = false;   // the combine's last CTA writes the status (no k_status launch)
        if (!s2 && npts > 0) s2 = combine_enqueue(h, dp, npts, dout, per_comp, &fused);
        if (!s2 && !fused && launch_status(h) != cudaSuccess) s2 = SGIGA_ERR_CUDA;
        h->cs_ready = false;
        if (h->cs_pending) {   // not consumed (an earlier step failed): still join the side stream
            cudaStreamWaitEvent(h->stream, h->cs_join, 0);
            h->cs_pending = false;
        }
        return s2;
    };
    // whole-run graph: only when the solve has no host-driven loop (every
    // component on the single-launch small path) and no profiling knob is on
    const bool can_graph = run_graphs_enabled(h) && h->large_comps.empty() && !h->graph_broken && !per_comp;
    const bool same = can_graph && h->rkey.npts == npts && h->rkey.rtol == rtol && h->rkey.maxit == maxit &&
                      h->rkey.dp == dp && h->rkey.dout == dout && h->rkey.hp == hsrc;
    if (same && h->run_exec) {
        SG_CUDA(cudaGraphLaunch(h->run_exec, h->stream));
        h->tables_ready = true;
        for (int i = 0; i < 3; ++i) h->launches[i] = h->run_launches[i];
        for (int i = 0; i < 7; ++i) h->kran[i] = h->run_kran[i];
        for (int i = 0; i < Handle::NEV; ++i) h->alias[i] = h->run_alias[i];
        h->last_mark = -1;
    } else if (same && h->rkey.warm) {
        cudaGraph_t g = nullptr;
        SG_CUDA(cudaStreamBeginCapture(h->stream, cudaStreamCaptureModeThreadLocal));
        h->capturing = true;
        st = enqueue_all();
        h->capturing = false;
        const cudaError_t ce = cudaStreamEndCapture(h->stream, &g);
        cudaError_t ie = cudaErrorUnknown;
        if (!st && ce == cudaSuccess && g) ie = cudaGraphInstantiate(&h->run_exec, g, 0);
        if (g) cudaGraphDestroy(g);
        if (st || ie != cudaSuccess) {   // not capturable here: run the launches directly from now on
            cudaGetLastError();
            h->run_exec = nullptr;
            h->drop_run_graph();
            h->graph_broken = true;
            if ((st = enqueue_all())) return st;
        } else {
            for (int i = 0; i < 3; ++i) h->run_launches[i] = h->launches[i];
            for (int i = 0; i < 7; ++i) h->run_kran[i] = h->kran[i];
            for (int i = 0; i < Handle::NEV; ++i) h->run_alias[i] = h->alias[i];
            h->last_mark = -1;
            SG_CUDA(cudaGraphLaunch(h->run_exec, h->stream));
        }
    } else {
        if ((st = enqueue_all())) return st;
        if (can_graph) {
            h->drop_run_graph();
            h->rkey.rtol = rtol; h->rkey.maxit = maxit; h->rkey.dp = dp; h->rkey.dout = dout; h->rkey.hp = hsrc;
            h->rkey.npts = npts; h->rkey.warm = 1;
        }
    }
    h->run_npts = npts;
    return SGIGA_OK;
}

// the one synchronisation of a pass and its verdict
static int run_finish(Handle* h, int32_t* iters_out, double* relres_out) {
    SG_CUDA(cudaStreamSynchronize(h->stream));
    // every pass since the last verdict OR-ed its failure into the sticky
    // word: a pipelined pass that failed before the last one is reported too
    const int sticky = *reinterpret_cast<volatile int*>(h->h_sticky);
    *h->h_sticky = 0;
    int st = decode_err(h);
    if (st) return st;
    SG_CUDA(h->elapsed(&h->ms[0], Handle::PHASE_EV + 0, Handle::PHASE_EV + 1));
    h->assembled = true;
    st = solve_finish(h, iters_out, relres_out);
    if (h->run_npts > 0) SG_CUDA(h->elapsed(&h->ms[2], Handle::PHASE_EV + 4, Handle::PHASE_EV + 5));
    if (!st && sticky) {
        set_error((sticky & 2) ? "an earlier pipelined pass raised a device error flag"
                               : "an earlier pipelined pass failed the solver acceptance (non-finite, not "
                                 "converged, or relative residual > 1e-10)");
        st = (sticky & 2) ? SGIGA_ERR_VALUE : SGIGA_ERR_SOLVE;
    }
    return st;
}

int sgiga_run(sgiga_handle* hh, double rtol, int32_t maxit, const double* pts, int64_t npts,
              double* out, int32_t device, int32_t* iters_out, double* relres_out) {
    Handle* h = reinterpret_cast<Handle*>(hh);
    if (!h || npts < 0 || (npts > 0 && (!pts || !out))) { set_error("null argument"); return SGIGA_ERR_VALUE; }
    if (device < 0) { set_error("sgiga_run: per-component output is not supported"); return SGIGA_ERR_VALUE; }
    const double* dp = pts;
    double* dout = out;
    const double* hsrc = nullptr;
    int st;
    if (npts > 0 && device == 0) {
        cudaPointerAttributes pa{};
        const bool pinned = cudaPointerGetAttributes(&pa, pts) == cudaSuccess && pa.type == cudaMemoryTypeHost;
        cudaGetLastError();
        if (pinned) {   // uploaded on the point-sort side stream inside the pass
            if ((st = ensure_scratch(h, &h->d_spts, &h->spts_cap, (size_t)npts * h->d))) return st;
            if ((st = ensure_scratch(h, &h->d_sout, &h->sout_cap, (size_t)npts))) return st;
            dp = h->d_spts;
            dout = h->d_sout;
            hsrc = pts;
        } else if ((st = stage_points(h, pts, npts, (size_t)npts, &dp, &dout))) {
            return st;
        }
    }
    if ((st = run_enqueue(h, rtol, maxit, dp, npts, dout, hsrc))) return st;
    if (npts > 0 && device == 0)
        SG_CUDA(cudaMemcpyAsync(out, dout, sizeof(double) * npts, cudaMemcpyDeviceToHost, h->stream));
    return run_finish(h, iters_out, relres_out);
}

int sgiga_run_async(sgiga_handle* hh, double rtol, int32_t maxit, const double* pts_dev, int64_t npts,
                    double* out_dev) {
    Handle* h = reinterpret_cast<Handle*>(hh);
    if (!h || npts < 0 || (npts > 0 && (!pts_dev || !out_dev))) { set_error("null argument"); return SGIGA_ERR_VALUE; }
    return run_enqueue(h, rtol, maxit, pts_dev, npts, out_dev);
}

int sgiga_run_components_async(sgiga_handle* hh, double rtol, int32_t maxit, const double* pts_dev, int64_t npts,
                               double* out_dev) {
    Handle* h = reinterpret_cast<Handle*>(hh);
    if (!h || npts < 0 || (npts > 0 && (!pts_dev || !out_dev))) { set_error("null argument"); return SGIGA_ERR_VALUE; }
    return run_enqueue(h, rtol, maxit, pts_dev, npts, out_dev, nullptr, 1);
}

int sgiga_run_host_async(sgiga_handle* hh, double rtol, int32_t maxit, const double* pts_pinned, int64_t npts,
                         double* out_pinned) {
    Handle* h = reinterpret_cast<Handle*>(hh);
    if (!h || npts < 0 || (npts > 0 && (!pts_pinned || !out_pinned))) { set_error("null argument"); return SGIGA_ERR_VALUE; }
    const double* dp = nullptr;
    double* dout = nullptr;
    int st;
    if (npts > 0) {
        for (const void* ptr : {static_cast<const void*>(pts_pinned), static_cast<const void*>(out_pinned)}) {
            cudaPointerAttributes pa{};
            const bool pinned = cudaPointerGetAttributes(&pa, ptr) == cudaSuccess && pa.type == cudaMemoryTypeHost;
            cudaGetLastError();
            if (!pinned) { set_error("sgiga_run_host_async: points and output must be page-locked host memory"); return SGIGA_ERR_VALUE; }
        }
        if ((st = ensure_scratch(h, &h->d_spts, &h->spts_cap, (size_t)npts * h->d))) return st;
        if ((st = ensure_scratch(h, &h->d_sout, &h->sout_cap, (size_t)npts))) return st;
        dp = h->d_spts;
        dout = h->d_sout;
    }
    // the H2D of the points runs on the point-sort side stream inside the pass
    // (ordered after the previous pass's combine by the pass's fork event);
    // the D2H of the values follows the combine on the handle's stream
    if ((st = run_enqueue(h, rtol, maxit, dp, npts, dout, npts > 0 ? pts_pinned : nullptr))) return st;
    if (npts > 0)
        SG_CUDA(cudaMemcpyAsync(out_pinned, dout, sizeof(double) * npts, cudaMemcpyDeviceToHost, h->stream));
    return SGIGA_OK;
}

int sgiga_run_wait(sgiga_handle* hh, int32_t* iters_out, double* relres_out) {
    Handle* h = reinterpret_cast<Handle*>(hh);
    if (!h) return SGIGA_ERR_VALUE;
    return run_finish(h, iters_out, relres_out);
}

int sgiga_iterations(sgiga_handle* hh, int32_t* iters) {
    Handle* h = reinterpret_cast<Handle*>(hh);
    if (!h || !iters) return SGIGA_ERR_VALUE;
    for (int c = 0; c < h->ncomp; ++c) iters[c] = h->iters[c];
    return SGIGA_OK;
}

int sgiga_coefficients(sgiga_handle* hh, double* out) {
    Handle* h = reinterpret_cast<Handle*>(hh);
    if (!h || !out) return SGIGA_ERR_VALUE;
    if (!h->have_coefs) { set_error("no coefficients: solve or set them first"); return SGIGA_ERR_STATE; }
    SG_CUDA(cudaMemcpyAsync(out, h->d_coef, sizeof(double) * h->total_dofs, cudaMemcpyDeviceToHost, h->stream));
    SG_CUDA(cudaStreamSynchronize(h->stream));
    return SGIGA_OK;
}

int sgiga_set_coefficients(sgiga_handle* hh, const double* full) {
    Handle* h = reinterpret_cast<Handle*>(hh);
    if (!h || !full) return SGIGA_ERR_VALUE;
    SG_CUDA(cudaMemcpyAsync(h->d_coef, full, sizeof(double) * h->total_dofs, cudaMemcpyHostToDevice, h->stream));
    SG_CUDA(cudaStreamSynchronize(h->stream));
    h->begin_call();
    int st = ensure_tables(h);
    if (st) return st;
    h->have_coefs = true;
    return SGIGA_OK;
}

int sgiga_combine_points(sgiga_handle* hh, const double* pts, int64_t npts, double* out,
                         int32_t device) {
    Handle* h = reinterpret_cast<Handle*>(hh);
    if (!h || npts < 0) return SGIGA_ERR_VALUE;
    if (!h->have_coefs) { set_error("combine before solve"); return SGIGA_ERR_STATE; }
    if (npts == 0) return SGIGA_OK;
    const int per_comp = device < 0;   // device = -1 / -2: per-component values (host / device)
    const bool dev_ptrs = device == 1 || device == -2;
    const size_t nout = per_comp ? (size_t)npts * h->ncomp : (size_t)npts;
    const double* dp = pts;
    double* dout = out;
    int st;
    if (!dev_ptrs && (st = stage_points(h, pts, npts, nout, &dp, &dout))) return st;
    h->begin_call();
    if ((st = combine_enqueue(h, dp, npts, dout, per_comp))) return st;
    if (!dev_ptrs) SG_CUDA(cudaMemcpyAsync(out, dout, sizeof(double) * nout, cudaMemcpyDeviceToHost, h->stream));
    if ((st = check_err(h))) return st;   // synchronises; points outside [0,1]^d are reported here
    SG_CUDA(h->elapsed(&h->ms[2], Handle::PHASE_EV + 4, Handle::PHASE_EV + 5));
    return SGIGA_OK;
}

int sgiga_combine_grid(sgiga_handle* hh, const double* pts_per_dir, const int64_t* npd,
                       int32_t comp, double* vals, double* grads) {
    Handle* h = reinterpret_cast<Handle*>(hh);
    if (!h || !pts_per_dir || !npd || !vals) return SGIGA_ERR_VALUE;
    if (!h->have_coefs) { set_error("combine before solve"); return SGIGA_ERR_STATE; }
    if (comp >= h->ncomp) { set_error("component index out of range"); return SGIGA_ERR_KEY; }
    int64_t N = 1, P = 0;
    for (int k = 0; k < h->d; ++k) { N *= npd[k]; P += npd[k]; }
    double *dp = nullptr, *dv = nullptr, *dg = nullptr;
    SG_CUDA(cudaMalloc(&dp, sizeof(double) * std::max<int64_t>(P, 1)));
    SG_CUDA(cudaMalloc(&dv, sizeof(double) * std::max<int64_t>(N, 1)));
    if (grads) SG_CUDA(cudaMalloc(&dg, sizeof(double) * std::max<int64_t>(N * h->d, 1)));
    SG_CUDA(cudaMemcpyAsync(dp, pts_per_dir, sizeof(double) * P, cudaMemcpyHostToDevice, h->stream));
    SG_CUDA(launch_combine_grid(h, dp, npd, comp, dv, dg));
    SG_CUDA(cudaMemcpyAsync(vals, dv, sizeof(double) * N, cudaMemcpyDeviceToHost, h->stream));
    if (grads) SG_CUDA(cudaMemcpyAsync(grads, dg, sizeof(double) * N * h->d, cudaMemcpyDeviceToHost, h->stream));
    SG_CUDA(cudaStreamSynchronize(h->stream));
    cudaFree(dp); cudaFree(dv);
    if (dg) cudaFree(dg);
    return SGIGA_OK;
}

static int error_norms_impl(Handle* h, const double* pts, const double* wts, const int64_t* npd,
                            int32_t nterm, const int32_t* tcomp, const double* tw, int32_t solution_id,
                            double* out) {
    if (!h->have_coefs) { set_error("error norms before solve"); return SGIGA_ERR_STATE; }
    for (int t = 0; t < nterm; ++t)
        if (tcomp[t] < 0 || tcomp[t] >= h->ncomp) { set_error("term component index out of range"); return SGIGA_ERR_KEY; }
    int64_t N = 1, P = 0;
    for (int k = 0; k < h->d; ++k) { N *= npd[k]; P += npd[k]; }
    int64_t nb = (N + 255) / 256;
    double *dp = nullptr, *dw = nullptr, *dpart = nullptr, *dtw = nullptr;
    int* dtc = nullptr;
    SG_CUDA(cudaMalloc(&dp, sizeof(double) * std::max<int64_t>(P, 1)));
    SG_CUDA(cudaMalloc(&dw, sizeof(double) * std::max<int64_t>(P, 1)));
    SG_CUDA(cudaMalloc(&dpart, sizeof(double) * (2 * nb + 2)));
    SG_CUDA(cudaMemcpyAsync(dp, pts, sizeof(double) * P, cudaMemcpyHostToDevice, h->stream));
    SG_CUDA(cudaMemcpyAsync(dw, wts, sizeof(double) * P, cudaMemcpyHostToDevice, h->stream));
    if (nterm > 0) {
        SG_CUDA(cudaMalloc(&dtc, sizeof(int) * nterm));
        SG_CUDA(cudaMalloc(&dtw, sizeof(double) * nterm));
        SG_CUDA(cudaMemcpyAsync(dtc, tcomp, sizeof(int) * nterm, cudaMemcpyHostToDevice, h->stream));
        SG_CUDA(cudaMemcpyAsync(dtw, tw, sizeof(double) * nterm, cudaMemcpyHostToDevice, h->stream));
    }
    int64_t nbl = 0;
    SG_CUDA(launch_error_norms(h, dp, dw, npd, solution_id, dpart, &nbl, dtc, dtw, nterm));
    SG_CUDA(cudaMemcpyAsync(out, dpart + 2 * nbl, 2 * sizeof(double), cudaMemcpyDeviceToHost, h->stream));
    SG_CUDA(cudaStreamSynchronize(h->stream));
    cudaFree(dp); cudaFree(dw); cudaFree(dpart);
    if (dtc) cudaFree(dtc);
    if (dtw) cudaFree(dtw);
    return check_err(h);
}

int sgiga_error_norms(sgiga_handle* hh, const double* pts, const double* wts,
                      const int64_t* npd, int32_t solution_id, double* out) {
    Handle* h = reinterpret_cast<Handle*>(hh);
    if (!h || !pts || !wts || !npd || !out) return SGIGA_ERR_VALUE;
    if (solution_id < 0) { set_error("unknown solution id"); return SGIGA_ERR_VALUE; }
    return error_norms_impl(h, pts, wts, npd, 0, nullptr, nullptr, solution_id, out);
}

int sgiga_subset_error_norms(sgiga_handle* hh, const double* pts, const double* wts,
                             const int64_t* npd, int32_t n_terms, const int32_t* comps,
                             const double* weights, int32_t solution_id, double* out) {
    Handle* h = reinterpret_cast<Handle*>(hh);
    if (!h || !pts || !wts || !npd || !out || n_terms < 1 || !comps || !weights) {
        set_error("null argument or empty term list");
        return SGIGA_ERR_VALUE;
    }
    return error_norms_impl(h, pts, wts, npd, n_terms, comps, weights, solution_id < 0 ? -1 : solution_id, out);
}

int sgiga_export_csr(sgiga_handle* hh, int32_t comp, int64_t* nnz_out, int64_t* indptr,
                     int32_t* indices, double* data, double* rhs) {
    Handle* h = reinterpret_cast<Handle*>(hh);
    if (!h || !nnz_out) return SGIGA_ERR_VALUE;
    if (comp < 0 || comp >= h->ncomp) { set_error("component index out of range"); return SGIGA_ERR_KEY; }
    if (!h->assembled) { set_error("export before assemble"); return SGIGA_ERR_STATE; }
    const CompInfo& C = h->comps[comp];
    const int d = h->d, p = h->p;
    std::vector<double> st((size_t)C.rows * C.nslots), b((size_t)C.rows);
    if (C.rows) {
        SG_CUDA(cudaMemcpy(st.data(), h->d_stencil + C.mat_off, sizeof(double) * st.size(), cudaMemcpyDeviceToHost));
        SG_CUDA(cudaMemcpy(b.data(), h->d_rhs + C.vec_off, sizeof(double) * b.size(), cudaMemcpyDeviceToHost));
    }
    int64_t M[3] = {1, 1, 1};
    for (int k = d - 2; k >= 0; --k) M[k] = M[k + 1] * C.m[k + 1];
    int64_t nnz = 0;
    if (indptr) indptr[0] = 0;
    for (int64_t ref = 0; ref < C.rows; ++ref) {
        int r[3] = {0, 0, 0};
        int64_t rem = ref, irow = 0;
        for (int k = d - 1; k >= 0; --k) { r[k] = (int)(rem % C.m[k]); rem /= C.m[k]; }
        for (int k = 0; k < d; ++k) irow += (int64_t)r[k] * C.rs[k];
        if (rhs) rhs[ref] = b[irow];
        int S0 = C.S[0], S1 = d > 1 ? C.S[1] : 1, S2 = d > 2 ? C.S[2] : 1;
        for (int s0 = 0; s0 < S0; ++s0)
            for (int s1 = 0; s1 < S1; ++s1)
                for (int s2 = 0; s2 < S2; ++s2) {
                    int sl[3] = {s0, s1, s2};
                    int64_t col = 0, slot = 0;
                    bool ok = true;
                    for (int k = 0; k < d; ++k) {
                        int c = C.absm[k] ? sl[k] : r[k] + sl[k] - p;
                        if (c < 0 || c >= C.m[k] || std::abs(c - r[k]) > p) { ok = false; break; }
                        col += (int64_t)c * M[k];
                        slot += (int64_t)sl[k] * C.ss[k];
                    }
                    if (!ok) continue;
                    double v = st[(size_t)slot * C.rows + irow];
                    if (v == 0.0) continue;   // scipy csr addition drops exact zeros
                    if (indices) indices[nnz] = (int32_t)col;
                    if (data) data[nnz] = v;
                    ++nnz;
                }
        if (indptr) indptr[ref + 1] = nnz;
    }
    *nnz_out = nnz;
    return SGIGA_OK;
}

int sgiga_basis_table(sgiga_handle* hh, int32_t axis, int32_t level, int32_t* nel_out, double* vals,
                      double* ders, double* pts, double* wts) {
    Handle* h = reinterpret_cast<Handle*>(hh);
    if (!h || !nel_out) { set_error("null argument"); return SGIGA_ERR_VALUE; }
    if (axis < 0 || axis >= h->d || level < 0 || level > h->max_level) {
        set_error("axis / level out of range");
        return SGIGA_ERR_VALUE;
    }
    const int t = h->tab_of[(size_t)axis * (h->max_level + 1) + level];
    if (t < 0) { set_error("no component of the plan uses this (axis, level)"); return SGIGA_ERR_KEY; }
    const TabInfo& T = h->tabs[t];
    *nel_out = T.nel;
    if (!vals && !ders && !pts && !wts) return SGIGA_OK;
    if (!h->assembled && !h->tables_ready) { set_error("basis tables before assembly"); return SGIGA_ERR_STATE; }
    SG_CUDA(cudaStreamSynchronize(h->stream));
    const size_t nv = (size_t)T.nel * h->q * (h->p + 1), nq = (size_t)T.nel * h->q;
    if (vals) SG_CUDA(cudaMemcpy(vals, h->d_tabvals + T.val_off, sizeof(double) * nv, cudaMemcpyDeviceToHost));
    if (ders) SG_CUDA(cudaMemcpy(ders, h->d_tabvals + T.val_off + nv, sizeof(double) * nv, cudaMemcpyDeviceToHost));
    if (pts) SG_CUDA(cudaMemcpy(pts, h->d_qx + T.qp_off, sizeof(double) * nq, cudaMemcpyDeviceToHost));
    if (wts) SG_CUDA(cudaMemcpy(wts, h->d_qw + T.qp_off, sizeof(double) * nq, cudaMemcpyDeviceToHost));
    return SGIGA_OK;
}

int sgiga_phase_stats(sgiga_handle* hh, float* ms3, int64_t* launches3) {
    Handle* h = reinterpret_cast<Handle*>(hh);
    if (!h) return SGIGA_ERR_VALUE;
    for (int i = 0; i < 3; ++i) {
        if (ms3) ms3[i] = h->ms[i];
        if (launches3) launches3[i] = h->launches[i];
    }
    return SGIGA_OK;
}

int sgiga_kernel_times(sgiga_handle* hh, float* ms7) {
    Handle* h = reinterpret_cast<Handle*>(hh);
    if (!h || !ms7) return SGIGA_ERR_VALUE;
    SG_CUDA(cudaStreamSynchronize(h->stream));
    for (int g = 0; g < 7; ++g) {
        float ms = 0.0f;
        if (h->kran[g] && h->elapsed(&ms, 2 * g, 2 * g + 1) != cudaSuccess) ms = -1.0f;
        ms7[g] = h->kran[g] ? ms : 0.0f;
    }
    cudaGetLastError();
    return SGIGA_OK;
}

int sgiga_assembly_flops(sgiga_handle* hh, double* executed) {
    Handle* h = reinterpret_cast<Handle*>(hh);
    if (!h || !executed) return SGIGA_ERR_VALUE;
    *executed = h->asm_tiled ? h->tiles3_flops : 0.0;
    return SGIGA_OK;
}

int sgiga_assembly_kind(sgiga_handle* hh, int32_t* kind) {
    Handle* h = reinterpret_cast<Handle*>(hh);
    if (!h || !kind) return SGIGA_ERR_VALUE;
    *kind = h->asm_tiled ? 1 : (h->box_state > 0 ? 2 : 0);
    return SGIGA_OK;
}

void* sgiga_stream(sgiga_handle* hh) {
    Handle* h = reinterpret_cast<Handle*>(hh);
    return h ? (void*)h->stream : nullptr;
}

int sgiga_destroy(sgiga_handle* hh) {
    Handle* h = reinterpret_cast<Handle*>(hh);
    if (!h) return SGIGA_OK;
    if (h->stream) cudaStreamSynchronize(h->stream);
    free_all(h);
    delete h;
    return SGIGA_OK;
}

}  // extern "C"
