// OptV2 building-block kernels of the reference API, one thread per triangle, SoA output
// (r x nme, row il contiguous = the reference's C-ordered Kg / Ig / Jg arrays):
//   batch_kg_mass/_mass_weighted/_stiff/_elastic  assembly.py:214-307
//   build_ig_jg_p1 / build_ig_jg_p1_vector         assembly.py:162-192
//   batch_gradients                                assembly.py:195-211
//   compute_areas                                  mesh.py:51-69
// These feed the batch_* Python API and the general TripletBatch.to_csc path; the fused
// assemble() path (fa_assembly.cu) never materialises Kg.
#include "fa_common.cuh"
#include "fa_element.cuh"

namespace fa {

template <int KIND>
__global__ void k_element_kg(const int32_t* __restrict__ me, int64_t nme, const double2* __restrict__ q,
                             const double* __restrict__ areas, const double* __restrict__ w, double lam, double mu,
                             double* __restrict__ kg, fa_result* res) {
    for (int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; k < nme; k += int64_t(gridDim.x) * blockDim.x) {
        const double area = areas[k];
        if (KIND != FA_KIND_MASSW && area <= AREA_EPS) atomic_min_i64(&res->degenerate_index, k);
        if constexpr (KIND == FA_KIND_MASS) {
            const MassTri t = mass_prepare(area);
#pragma unroll
            for (int il = 0; il < 9; ++il) kg[il * nme + k] = (il % 4 == 0) ? t.d : t.o;
        } else if constexpr (KIND == FA_KIND_MASSW) {
            const int c0 = me[3 * k], c1 = me[3 * k + 1], c2 = me[3 * k + 2];
            const MasswTri t = massw_prepare(area, w[c0], w[c1], w[c2]);
#pragma unroll
            for (int il = 0; il < 9; ++il) kg[il * nme + k] = massw_entry(t, il % 3, il / 3);
        } else if constexpr (KIND == FA_KIND_STIFF) {
            const int c0 = me[3 * k], c1 = me[3 * k + 1], c2 = me[3 * k + 2];
            const StiffTri t = stiff_prepare(q[c0], q[c1], q[c2], area);
            // rows 0,1,2,4,5,8 computed, 3,6,7 copies of 1,2,5 (assembly.py:257-263)
            const double k0 = stiff_entry(t, 0, 0), k1 = stiff_entry(t, 1, 0), k2 = stiff_entry(t, 2, 0);
            const double k4 = stiff_entry(t, 1, 1), k5 = stiff_entry(t, 2, 1), k8 = stiff_entry(t, 2, 2);
            kg[0 * nme + k] = k0; kg[1 * nme + k] = k1; kg[2 * nme + k] = k2;
            kg[3 * nme + k] = k1; kg[4 * nme + k] = k4; kg[5 * nme + k] = k5;
            kg[6 * nme + k] = k2; kg[7 * nme + k] = k5; kg[8 * nme + k] = k8;
        } else {
            const int c0 = me[3 * k], c1 = me[3 * k + 1], c2 = me[3 * k + 2];
            const ElasticTri t = elastic_prepare(q[c0], q[c1], q[c2], area);
            const double P = FADD(lam, FMUL(2.0, mu));
#pragma unroll
            for (int r = 0; r < 36; ++r) kg[r * nme + k] = elastic_entry(t, r % 6, r / 6, lam, mu, P);
        }
    }
}

// Element-loop strategies (assembly.py:359-397): every triangle's element matrix from the
// per-element formulas of elements.py, as triplets in triangle-major order (position k*r + il,
// il = a + order*b, the ravel(order="F") of _assemble_triplet_loop, assembly.py:377-397).
template <int KIND>
__global__ void k_element_triplets(const int32_t* __restrict__ me, int64_t nme, const double2* __restrict__ q,
                                   const double* __restrict__ areas, const double* __restrict__ w, double lam,
                                   double mu, int64_t* __restrict__ rows, int64_t* __restrict__ cols,
                                   double* __restrict__ vals, fa_result* res) {
    constexpr int ORD = KIND == FA_KIND_ELASTIC ? 6 : 3;
    constexpr int R = ORD * ORD;
    for (int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; k < nme; k += int64_t(gridDim.x) * blockDim.x) {
        const double area = areas[k];
        if (!(area > AREA_EPS)) atomic_min_i64(&res->degenerate_index, k);  // _check_area (elements.py:27-31)
        const int c[3] = {me[3 * k], me[3 * k + 1], me[3 * k + 2]};
        const bool need_q = KIND == FA_KIND_STIFF || KIND == FA_KIND_ELASTIC;
        const double2 p1 = need_q ? q[c[0]] : make_double2(0.0, 0.0);
        const double2 p2 = need_q ? q[c[1]] : make_double2(0.0, 0.0);
        const double2 p3 = need_q ? q[c[2]] : make_double2(0.0, 0.0);
        const bool need_w = KIND == FA_KIND_MASSW;
        ElemLoopTri m;
        elem_loop_matrix<KIND>(p1, p2, p3, area, need_w ? w[c[0]] : 0.0, need_w ? w[c[1]] : 0.0,
                               need_w ? w[c[2]] : 0.0, lam, mu, m);
        int64_t ids[ORD];
#pragma unroll
        for (int i = 0; i < ORD; ++i) ids[i] = ORD == 3 ? int64_t(c[i]) : 2 * int64_t(c[i / 2]) + (i & 1);
#pragma unroll
        for (int b = 0; b < ORD; ++b)
#pragma unroll
            for (int a = 0; a < ORD; ++a) {
                const int64_t o = k * R + a + ORD * b;
                rows[o] = ids[a];
                cols[o] = ids[b];
                vals[o] = m.e[a][b];
            }
    }
}

__global__ void k_ig_jg(const int32_t* __restrict__ me, int64_t nme, int vector, int32_t* __restrict__ ig,
                        int32_t* __restrict__ jg) {
    for (int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; k < nme; k += int64_t(gridDim.x) * blockDim.x) {
        const int32_t c[3] = {me[3 * k], me[3 * k + 1], me[3 * k + 2]};
        if (!vector) {
#pragma unroll
            for (int il = 0; il < 9; ++il) {
                ig[il * nme + k] = c[il % 3];
                jg[il * nme + k] = c[il / 3];
            }
        } else {
            // dofs (2*i1, 2*i1+1, 2*i2, 2*i2+1, 2*i3, 2*i3+1) (assembly.py:186-189)
#pragma unroll
            for (int il = 0; il < 36; ++il) {
                const int a = il % 6, b = il / 6;
                ig[il * nme + k] = 2 * c[a / 2] + (a & 1);
                jg[il * nme + k] = 2 * c[b / 2] + (b & 1);
            }
        }
    }
}

__global__ void k_gradients(const int32_t* __restrict__ me, int64_t nme, const double2* __restrict__ q,
                            const double* __restrict__ areas, double* __restrict__ g, fa_result* res) {
    for (int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; k < nme; k += int64_t(gridDim.x) * blockDim.x) {
        const double area = areas[k];
        if (area <= AREA_EPS) atomic_min_i64(&res->degenerate_index, k);
        const int c0 = me[3 * k], c1 = me[3 * k + 1], c2 = me[3 * k + 2];
        const ElasticTri t = elastic_prepare(q[c0], q[c1], q[c2], area);
        g[0 * nme + k] = t.g0.x; g[1 * nme + k] = t.g0.y;
        g[2 * nme + k] = t.g1.x; g[3 * nme + k] = t.g1.y;
        g[4 * nme + k] = t.g2.x; g[5 * nme + k] = t.g2.y;
    }
}

__global__ void k_areas(const int32_t* __restrict__ me, int64_t nme, const double2* __restrict__ q,
                        double* __restrict__ areas, fa_result* res) {
    for (int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; k < nme; k += int64_t(gridDim.x) * blockDim.x) {
        const double a = tri_area(q[me[3 * k]], q[me[3 * k + 1]], q[me[3 * k + 2]]);
        areas[k] = a;
        if (a <= AREA_EPS) atomic_min_i64(&res->degenerate_index, k);
    }
}

// Mesh ingestion (femasm Mesh.__init__, mesh.py:84-119, and compute_areas, mesh.py:51-69) in one
// pass over the int64 connectivity: range check (first bad flattened position), repeated ids
// (first triangle), int32 copy for the assembly plans, areas (bitwise compute_areas) and the first
// degenerate triangle.  Triangles with a bad id get area 0 and are not reported as degenerate
// (the reference raises the range / repeat errors first).
__global__ void k_ingest(const int64_t* __restrict__ me64, int64_t nme, int64_t nq, const double2* __restrict__ q,
                         int32_t* __restrict__ me32, double* __restrict__ areas, fa_result* res) {
    for (int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; k < nme; k += int64_t(gridDim.x) * blockDim.x) {
        const int64_t c0 = me64[3 * k], c1 = me64[3 * k + 1], c2 = me64[3 * k + 2];
        const bool r0 = c0 >= 0 && c0 < nq, r1 = c1 >= 0 && c1 < nq, r2 = c2 >= 0 && c2 < nq;
        if (!r0) atomic_min_i64(&res->index_error_pos, 3 * k);
        else if (!r1) atomic_min_i64(&res->index_error_pos, 3 * k + 1);
        else if (!r2) atomic_min_i64(&res->index_error_pos, 3 * k + 2);
        if (c0 == c1 || c1 == c2 || c0 == c2) atomic_min_i64(&res->repeat_error_pos, k);
        me32[3 * k] = int32_t(c0);
        me32[3 * k + 1] = int32_t(c1);
        me32[3 * k + 2] = int32_t(c2);
        double a = 0.0;
        if (r0 && r1 && r2) {
            a = tri_area(q[c0], q[c1], q[c2]);
            if (a <= AREA_EPS) atomic_min_i64(&res->degenerate_index, k);
        }
        areas[k] = a;
    }
}

}  // namespace fa

using namespace fa;

extern "C" int fa_mesh_ingest(const int64_t* d_me64, int64_t nme, int64_t nq, const double* d_q, int32_t* d_me32,
                              double* d_areas, fa_result* d_res, void* stream) {
    if (nme < 0 || nq < 1 || !d_me64 || !d_q || !d_me32 || !d_areas || !d_res) {
        set_error("fa_mesh_ingest: bad argument"); return FA_ERR_ARGUMENT;
    }
    if (nq > INT32_MAX) { set_error("fa_mesh_ingest: nq=%lld beyond 32-bit vertex ids", (long long)nq); return FA_ERR_TOO_LARGE; }
    cudaStream_t st = as_stream(stream);
    k_result_reset<<<1, 32, 0, st>>>(d_res);
    if (nme == 0) return FA_OK;
    const int tb = 256;
    k_ingest<<<grid_for(nme, tb), tb, 0, st>>>(d_me64, nme, nq, reinterpret_cast<const double2*>(d_q), d_me32, d_areas, d_res);
    FA_LAUNCH_CHECK("k_ingest");
    return FA_OK;
}

extern "C" int fa_element_kg(int kind, const int32_t* d_me, int64_t nme, const double* d_q, const double* d_areas,
                             const double* d_w, double lam, double mu, double* d_kg, fa_result* d_res, void* stream) {
    if (kind < 0 || kind > 3) { set_error("unknown matrix kind %d", kind); return FA_ERR_ARGUMENT; }
    if (nme < 0 || !d_kg || !d_areas || !d_res) { set_error("fa_element_kg: bad argument"); return FA_ERR_ARGUMENT; }
    if (kind != FA_KIND_MASS && !d_me) { set_error("fa_element_kg: connectivity required"); return FA_ERR_ARGUMENT; }
    if ((kind == FA_KIND_STIFF || kind == FA_KIND_ELASTIC) && !d_q) { set_error("fa_element_kg: coordinates required"); return FA_ERR_ARGUMENT; }
    if (kind == FA_KIND_MASSW && !d_w) { set_error("WEIGHTED_MASS requires a WeightField"); return FA_ERR_ARGUMENT; }
    cudaStream_t st = as_stream(stream);
    k_result_reset<<<1, 32, 0, st>>>(d_res);
    if (nme == 0) return FA_OK;
    const int tb = 256, gb = grid_for(nme, tb);
    const double2* q = reinterpret_cast<const double2*>(d_q);
    switch (kind) {
        case FA_KIND_MASS: k_element_kg<FA_KIND_MASS><<<gb, tb, 0, st>>>(d_me, nme, q, d_areas, d_w, lam, mu, d_kg, d_res); break;
        case FA_KIND_MASSW: k_element_kg<FA_KIND_MASSW><<<gb, tb, 0, st>>>(d_me, nme, q, d_areas, d_w, lam, mu, d_kg, d_res); break;
        case FA_KIND_STIFF: k_element_kg<FA_KIND_STIFF><<<gb, tb, 0, st>>>(d_me, nme, q, d_areas, d_w, lam, mu, d_kg, d_res); break;
        default: k_element_kg<FA_KIND_ELASTIC><<<gb, tb, 0, st>>>(d_me, nme, q, d_areas, d_w, lam, mu, d_kg, d_res); break;
    }
    FA_LAUNCH_CHECK("k_element_kg");
    return FA_OK;
}

extern "C" int fa_element_triplets(int kind, const int32_t* d_me, int64_t nme, const double* d_q, const double* d_areas,
                                   const double* d_w, double lam, double mu, int64_t* d_rows, int64_t* d_cols,
                                   double* d_vals, fa_result* d_res, void* stream) {
    if (kind < 0 || kind > 3) { set_error("unknown matrix kind %d", kind); return FA_ERR_ARGUMENT; }
    if (nme < 0 || !d_me || !d_areas || !d_rows || !d_cols || !d_vals || !d_res) {
        set_error("fa_element_triplets: bad argument"); return FA_ERR_ARGUMENT;
    }
    if ((kind == FA_KIND_STIFF || kind == FA_KIND_ELASTIC) && !d_q) { set_error("fa_element_triplets: coordinates required"); return FA_ERR_ARGUMENT; }
    if (kind == FA_KIND_MASSW && !d_w) { set_error("WEIGHTED_MASS requires a WeightField"); return FA_ERR_ARGUMENT; }
    cudaStream_t st = as_stream(stream);
    k_result_reset<<<1, 32, 0, st>>>(d_res);
    if (nme == 0) return FA_OK;
    const int tb = 128, gb = grid_for(nme, tb);
    const double2* q = reinterpret_cast<const double2*>(d_q);
    switch (kind) {
        case FA_KIND_MASS: k_element_triplets<FA_KIND_MASS><<<gb, tb, 0, st>>>(d_me, nme, q, d_areas, d_w, lam, mu, d_rows, d_cols, d_vals, d_res); break;
        case FA_KIND_MASSW: k_element_triplets<FA_KIND_MASSW><<<gb, tb, 0, st>>>(d_me, nme, q, d_areas, d_w, lam, mu, d_rows, d_cols, d_vals, d_res); break;
        case FA_KIND_STIFF: k_element_triplets<FA_KIND_STIFF><<<gb, tb, 0, st>>>(d_me, nme, q, d_areas, d_w, lam, mu, d_rows, d_cols, d_vals, d_res); break;
        default: k_element_triplets<FA_KIND_ELASTIC><<<gb, tb, 0, st>>>(d_me, nme, q, d_areas, d_w, lam, mu, d_rows, d_cols, d_vals, d_res); break;
    }
    FA_LAUNCH_CHECK("k_element_triplets");
    return FA_OK;
}

extern "C" int fa_build_ig_jg(int vector, const int32_t* d_me, int64_t nme, int32_t* d_ig, int32_t* d_jg, void* stream) {
    if (nme < 0 || !d_me || !d_ig || !d_jg) { set_error("fa_build_ig_jg: bad argument"); return FA_ERR_ARGUMENT; }
    if (nme == 0) return FA_OK;
    const int tb = 256;
    k_ig_jg<<<grid_for(nme, tb), tb, 0, as_stream(stream)>>>(d_me, nme, vector ? 1 : 0, d_ig, d_jg);
    FA_LAUNCH_CHECK("k_ig_jg");
    return FA_OK;
}

extern "C" int fa_batch_gradients(const int32_t* d_me, int64_t nme, const double* d_q, const double* d_areas,
                                  double* d_g, fa_result* d_res, void* stream) {
    if (nme < 0 || !d_me || !d_q || !d_areas || !d_g || !d_res) { set_error("fa_batch_gradients: bad argument"); return FA_ERR_ARGUMENT; }
    cudaStream_t st = as_stream(stream);
    k_result_reset<<<1, 32, 0, st>>>(d_res);
    if (nme == 0) return FA_OK;
    const int tb = 256;
    k_gradients<<<grid_for(nme, tb), tb, 0, st>>>(d_me, nme, reinterpret_cast<const double2*>(d_q), d_areas, d_g, d_res);
    FA_LAUNCH_CHECK("k_gradients");
    return FA_OK;
}

extern "C" int fa_compute_areas(const int32_t* d_me, int64_t nme, const double* d_q, double* d_areas, fa_result* d_res,
                                void* stream) {
    if (nme < 0 || !d_me || !d_q || !d_areas || !d_res) { set_error("fa_compute_areas: bad argument"); return FA_ERR_ARGUMENT; }
    cudaStream_t st = as_stream(stream);
    k_result_reset<<<1, 32, 0, st>>>(d_res);
    if (nme == 0) return FA_OK;
    const int tb = 256;
    k_areas<<<grid_for(nme, tb), tb, 0, st>>>(d_me, nme, reinterpret_cast<const double2*>(d_q), d_areas, d_res);
    FA_LAUNCH_CHECK("k_areas");
    return FA_OK;
}
