// unit_kernels.cu — unit-level entry points of the hot-path pieces, used by
// the parity tests against the reference's own QP / barrier tests:
//   mrsim_qp_solve_batch      <- solve_qp (qp.hpp:183-357), one warp per QP
//   mrsim_apply_barrier_batch <- apply_barrier (barrier.hpp:132-205), one group per team
// Both run the same device code as the fused step kernel (qp_solve_group,
// barrier_filter).
#include <cstring>
#include <vector>

#include "launch.h"
#include "mrsim_cuda.h"

namespace mrsim_dev {

constexpr int kQpMaxN = 32;
constexpr int kQpMaxM = 64;

// one problem's smem: the QP workspace, then G [m][n], h [m], u scratch, lo, hi [n] (each 16-byte aligned)
template <class Real>
__host__ __device__ constexpr int qp_slot_bytes(int n, int m) {
    typedef typename DenseRows<Real, 16, kQpMaxM>::Desc D;
    return ((QpWs<Real, D>::bytes(n) + 15) & ~15) + (((m * n + m + 3 * n) * static_cast<int>(sizeof(Real)) + 15) & ~15);
}

template <class Real>
__global__ void __launch_bounds__(32) qp_batch_kernel(int count, int n, int m, const double* A, const double* b,
                                                      const double* lo, const double* hi, const double* unom,
                                                      double tol, double* u_out, int32_t* status_out,
                                                      int32_t* iters_out) {
    // one warp = two problems (16 lanes each, lane l owns variables 2l, 2l+1)
    constexpr int L = 16;
    extern __shared__ __align__(16) unsigned char qsmem[];
    const Grp<L> g;
    const int lane = g.lane;
    const int slot = threadIdx.x / L;
    typedef typename DenseRows<Real, L, kQpMaxM>::Desc DDesc;
    unsigned char* sbase = qsmem + slot * qp_slot_bytes<Real>(n, m);
    QpWs<Real, DDesc> ws;
    ws.carve(sbase, n);
    Real* Gs = reinterpret_cast<Real*>(sbase + ((QpWs<Real, DDesc>::bytes(n) + 15) & ~15));
    Real* hs = Gs + m * n;
    Real* ushs = hs + m;
    Real* loss = ushs + n;
    Real* hiss = loss + n;
    const int t_real = blockIdx.x * 2 + slot;
    const bool ghost = t_real >= count;
    const int t = ghost ? count - 1 : t_real;
    const double* At = A + static_cast<size_t>(t) * m * n;
    // fold_rows (qp.hpp:104-141): normalise; zero rows keep b unnormalised
    for (int r = lane; r < m; r += L) {
        double norm = 0.0;
        for (int i = 0; i < n; ++i) norm += At[r * n + i] * At[r * n + i];
        norm = sqrt(norm);
        const double br = b[static_cast<size_t>(t) * m + r];
        if (norm < 1e-14) {
            for (int i = 0; i < n; ++i) Gs[r * n + i] = Real(0);
            hs[r] = Real(br);
        } else {
            for (int i = 0; i < n; ++i) Gs[r * n + i] = Real(At[r * n + i] / norm);
            hs[r] = Real(br / norm);
        }
    }
    for (int v = lane; v < n; v += L) {
        loss[v] = Real(lo[static_cast<size_t>(t) * n + v]);
        hiss[v] = Real(hi[static_cast<size_t>(t) * n + v]);
    }
    Grp<L>::sync();
    int boxes = 0;
    for (int i = 0; i < n; ++i) {
        boxes += hi[static_cast<size_t>(t) * n + i] < 1e30 ? 1 : 0;
        boxes += lo[static_cast<size_t>(t) * n + i] > -1e30 ? 1 : 0;
    }
    DenseRows<Real, L, kQpMaxM> rows{Gs, hs, ushs, loss, hiss, n, m, 0ull, 0ull};
    const bool vl = 2 * lane < n;
    Real ux = vl ? Real(unom[static_cast<size_t>(t) * n + 2 * lane]) : Real(0);
    Real uy = (vl && 2 * lane + 1 < n) ? Real(unom[static_cast<size_t>(t) * n + 2 * lane + 1]) : Real(0);
    const int status = qp_solve<Real, L>(g, rows, ws, n, !ghost, ux, uy, m + boxes, Real(tol));
    if (!ghost) {
        if (vl) u_out[static_cast<size_t>(t) * n + 2 * lane] = double(ux);
        if (vl && 2 * lane + 1 < n) u_out[static_cast<size_t>(t) * n + 2 * lane + 1] = double(uy);
        if (lane == 0) {
            status_out[t] = status;
            iters_out[t] = 0;
        }
    }
}

template <class Real, int L>
__global__ void __launch_bounds__(128) barrier_batch_kernel(const __grid_constant__ mrsim_cfg c, PhysConsts<Real> k,
                                                            int count, int N, const double* poses,
                                                            const double* nominal, int nobs, const double* obstacles,
                                                            const uint64_t* masks, double* cmds, int32_t* infeasible,
                                                            int32_t* coincident, int smem_group) {
    constexpr int MP = LaneCfg<L>::kMaxPair;  // any N <= L
    constexpr int MO = MRSIM_MAX_SLOTS;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const Grp<L> g;
    const int lane = g.lane;
    const int gib = threadIdx.x / L;
    const long long t_real = static_cast<long long>(blockIdx.x) * (blockDim.x / L) + gib;
    const bool ghost = t_real >= count;
    const long long t = ghost ? count - 1 : t_real;
    const int n = 2 * N, P = N * (N - 1) / 2;
    QpWs<Real, BarrierDesc<Real>> ws;
    ws.carve(smem_raw + gib * smem_group, n);
    Real* rcache = reinterpret_cast<Real*>(smem_raw + gib * smem_group +
                                           ((QpWs<Real, BarrierDesc<Real>>::bytes(n) + 15) & ~15));
    const bool vl = lane < N;
    const int ri = vl ? lane : 0;
    const double* ps = poses + t * N * 3;
    const double* nm = nominal + t * N * 2;
    const Real x = Real(ps[3 * ri]), y = Real(ps[3 * ri + 1]), th = Real(ps[3 * ri + 2]);
    const Real nv = dclamp(Real(nm[2 * ri]), -k.v_max, k.v_max);  // clamp_command (barrier.hpp:142)
    const Real nw = dclamp(Real(nm[2 * ri + 1]), -k.w_max, k.w_max);
    Real cv = nv, cw = nw;
    int status = kQpOptimal;
    if (c.barrier_enabled) {
        BarrierRows<Real, L, MP, MO> rows;
        __shared__ unsigned char pair_tab[MRSIM_MAX_ROBOTS * (MRSIM_MAX_ROBOTS - 1)];
        init_rows(rows, rcache, pair_tab, lane, N, k.cap);
        rows.oxy = obstacles + t * nobs * 3;  // (x, y, r) per obstacle
        rows.orad = rows.oxy + 2;
        rows.ostride = 3;
        rows.oinfl = c.projection_distance + c.discrete_margin;
        // static obstacles with masks (barrier.hpp:106-119), radius inflated (barrier.hpp:157)
        int obs_rows = 0;
        for (int o = 0; o < nobs; ++o) {
            const uint64_t mk = masks ? masks[t * nobs + o] : 0ull;
            for (int i = 0; i < N; ++i) {
                if (mk != 0 && ((mk >> i) & 1ull) == 0) continue;
                ++obs_rows;
                if (vl && i == ri) {
#pragma unroll
                    for (int q = 0; q < MO; ++q)
                        if (q == rows.nob) {
                            rows.oslot[q] = o;
                        }
                    ++rows.nob;
                }
            }
        }
        Real sn, cs;
        dsincos(th, &sn, &cs);
        const Real prx = x + cs * k.l, pry = y + sn * k.l;
        status = barrier_filter<Real, L, MP, MO, true>(g, rows, ws, k, !ghost, prx, pry, cs, sn, nv, nw, P + 8 * N + obs_rows, cv,
                                         cw);
    }
    if (!ghost) {
        if (vl) {
            cmds[(t * N + ri) * 2] = double(cv);
            cmds[(t * N + ri) * 2 + 1] = double(cw);
        }
        if (lane == 0) {
            infeasible[t] = status == kQpInfeasible ? 1 : 0;
            coincident[t] = status < 0 ? 1 : 0;
        }
    }
}

// FMA-chain probe: 8 independent chains per thread, ITERS iterations.
template <class Real>
__global__ void __launch_bounds__(256) fma_probe_kernel(Real* out, int iters, Real a, Real b) {
    Real x[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = Real(threadIdx.x + k) * Real(1e-3);
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) x[k] = fma(x[k], a, b);
    }
    Real s = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += x[k];
    if (s == Real(12345.678)) out[0] = s;  // keep the chains live
}

}  // namespace mrsim_dev

namespace {

struct DevBuf {
    void* p = nullptr;
    ~DevBuf() { cudaFree(p); }
};

template <class T>
cudaError_t upload(DevBuf& d, const T* h, size_t count) {
    cudaError_t e = cudaMalloc(&d.p, sizeof(T) * (count > 0 ? count : 1));
    if (e != cudaSuccess || count == 0 || !h) return e;
    return cudaMemcpy(d.p, h, sizeof(T) * count, cudaMemcpyHostToDevice);
}

template <class Real, int L>
cudaError_t run_barrier(const mrsim_cfg& c, int count, const double* dp, const double* dn, int nobs,
                        const double* dobs, const uint64_t* dm, double* dc, int32_t* di, int32_t* dco) {
    mrsim_dev::PhysConsts<Real> k;
    mrsim_host::fill_consts(c, k);
    const int N = c.num_robots;
    const int block = 128;
    const int gpb = block / L;
    constexpr int MP = mrsim_dev::LaneCfg<L>::kMaxPair;
    const int sg = (((mrsim_dev::QpWs<Real, mrsim_dev::BarrierDesc<Real>>::bytes(2 * N) + 15) & ~15) +
                    mrsim_dev::GroupSmem<Real>::rc_reals(L, MP, MRSIM_MAX_SLOTS) * static_cast<int>(sizeof(Real)) + 15) &
                   ~15;
    const int grid = (count + gpb - 1) / gpb;
    auto kern = mrsim_dev::barrier_batch_kernel<Real, L>;
    if (sg * gpb > 46 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, sg * gpb);
    kern<<<grid, block, sg * gpb>>>(c, k, count, N, dp, dn, nobs, dobs, dm, dc, di, dco, sg);
    return cudaGetLastError();
}

}  // namespace

extern "C" {

double mrsim_probe_fma_peak(int device, int fp64) {
    if (cudaSetDevice(device) != cudaSuccess) return -1.0;
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    void* out = nullptr;
    cudaMalloc(&out, 16);
    const int iters = 1 << 14, block = 256, grid = sms * 8;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int rep = 0; rep < 4; ++rep) {
        cudaEventRecord(e0);
        if (fp64)
            mrsim_dev::fma_probe_kernel<double><<<grid, block>>>(static_cast<double*>(out), iters, 0.999999, 1e-7);
        else
            mrsim_dev::fma_probe_kernel<float><<<grid, block>>>(static_cast<float*>(out), iters, 0.999999f, 1e-7f);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        if (rep > 0 && ms < best) best = ms;
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(out);
    if (cudaGetLastError() != cudaSuccess) return -1.0;
    const double flops = 2.0 * 8.0 * iters * static_cast<double>(grid) * block;
    return flops / (best * 1e-3);
}

int mrsim_qp_solve_batch(int device, int fp64, int count, int n, int m, const double* A, const double* b,
                         const double* lo, const double* hi, const double* u_nom, double tolerance, double* u_out,
                         int32_t* status_out, int32_t* iterations_out) {
    if (count < 1 || n < 1 || n > mrsim_dev::kQpMaxN || m < 0 || m > mrsim_dev::kQpMaxM)
        return MRSIM_E_INVALID_ARGUMENT;
    if (cudaSetDevice(device) != cudaSuccess) return MRSIM_E_CUDA;
    DevBuf dA, db, dlo, dhi, du, dout, dst, dit;
    if ((upload(dA, A, static_cast<size_t>(count) * m * n)) != cudaSuccess) return MRSIM_E_CUDA;
    if ((upload(db, b, static_cast<size_t>(count) * m)) != cudaSuccess) return MRSIM_E_CUDA;
    if ((upload(dlo, lo, static_cast<size_t>(count) * n)) != cudaSuccess) return MRSIM_E_CUDA;
    if ((upload(dhi, hi, static_cast<size_t>(count) * n)) != cudaSuccess) return MRSIM_E_CUDA;
    if ((upload(du, u_nom, static_cast<size_t>(count) * n)) != cudaSuccess) return MRSIM_E_CUDA;
    if ((upload<double>(dout, nullptr, static_cast<size_t>(count) * n)) != cudaSuccess) return MRSIM_E_CUDA;
    if ((upload<int32_t>(dst, nullptr, count)) != cudaSuccess) return MRSIM_E_CUDA;
    if ((upload<int32_t>(dit, nullptr, count)) != cudaSuccess) return MRSIM_E_CUDA;
    const size_t smem_d = 2 * static_cast<size_t>(mrsim_dev::qp_slot_bytes<double>(n, m));
    const size_t smem_f = 2 * static_cast<size_t>(mrsim_dev::qp_slot_bytes<float>(n, m));
    if (smem_d > 48 * 1024)
        cudaFuncSetAttribute(mrsim_dev::qp_batch_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(smem_d));
    if (smem_f > 48 * 1024)
        cudaFuncSetAttribute(mrsim_dev::qp_batch_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(smem_f));
    if (fp64)
        mrsim_dev::qp_batch_kernel<double><<<(count + 1) / 2, 32, smem_d>>>(
            count, n, m, static_cast<double*>(dA.p), static_cast<double*>(db.p), static_cast<double*>(dlo.p),
            static_cast<double*>(dhi.p), static_cast<double*>(du.p), tolerance, static_cast<double*>(dout.p),
            static_cast<int32_t*>(dst.p), static_cast<int32_t*>(dit.p));
    else
        mrsim_dev::qp_batch_kernel<float><<<(count + 1) / 2, 32, smem_f>>>(
            count, n, m, static_cast<double*>(dA.p), static_cast<double*>(db.p), static_cast<double*>(dlo.p),
            static_cast<double*>(dhi.p), static_cast<double*>(du.p), tolerance, static_cast<double*>(dout.p),
            static_cast<int32_t*>(dst.p), static_cast<int32_t*>(dit.p));
    if (cudaDeviceSynchronize() != cudaSuccess) return MRSIM_E_CUDA;
    cudaMemcpy(u_out, dout.p, sizeof(double) * count * n, cudaMemcpyDeviceToHost);
    cudaMemcpy(status_out, dst.p, sizeof(int32_t) * count, cudaMemcpyDeviceToHost);
    if (iterations_out) cudaMemcpy(iterations_out, dit.p, sizeof(int32_t) * count, cudaMemcpyDeviceToHost);
    return cudaGetLastError() == cudaSuccess ? MRSIM_OK : MRSIM_E_CUDA;
}

int mrsim_apply_barrier_batch(int device, int fp64, const mrsim_cfg* cfg, int count, const double* poses,
                              const double* nominal, int num_obstacles, const double* obstacles,
                              const uint64_t* obstacle_masks, double* commands_out, int32_t* infeasible_out) {
    if (!cfg || count < 1 || num_obstacles < 0 || num_obstacles > MRSIM_MAX_SLOTS) return MRSIM_E_INVALID_ARGUMENT;
    const int N = cfg->num_robots;
    if (N < 1 || N > MRSIM_MAX_ROBOTS) return MRSIM_E_UNSUPPORTED;
    if (cudaSetDevice(device) != cudaSuccess) return MRSIM_E_CUDA;
    DevBuf dp, dn, dobs, dm, dc, di, dco;
    if (upload(dp, poses, static_cast<size_t>(count) * N * 3) != cudaSuccess) return MRSIM_E_CUDA;
    if (upload(dn, nominal, static_cast<size_t>(count) * N * 2) != cudaSuccess) return MRSIM_E_CUDA;
    if (upload(dobs, obstacles, static_cast<size_t>(count) * num_obstacles * 3) != cudaSuccess) return MRSIM_E_CUDA;
    if (upload(dm, obstacle_masks, static_cast<size_t>(count) * num_obstacles) != cudaSuccess) return MRSIM_E_CUDA;
    if (upload<double>(dc, nullptr, static_cast<size_t>(count) * N * 2) != cudaSuccess) return MRSIM_E_CUDA;
    if (upload<int32_t>(di, nullptr, count) != cudaSuccess) return MRSIM_E_CUDA;
    if (upload<int32_t>(dco, nullptr, count) != cudaSuccess) return MRSIM_E_CUDA;
    const double* P_ = static_cast<double*>(dp.p);
    const double* N_ = static_cast<double*>(dn.p);
    const double* O_ = static_cast<double*>(dobs.p);
    const uint64_t* M_ = obstacle_masks ? static_cast<uint64_t*>(dm.p) : nullptr;
    double* C_ = static_cast<double*>(dc.p);
    int32_t* I_ = static_cast<int32_t*>(di.p);
    int32_t* X_ = static_cast<int32_t*>(dco.p);
    cudaError_t e;
    if (fp64) {
        if (N <= 4) e = run_barrier<double, 4>(*cfg, count, P_, N_, num_obstacles, O_, M_, C_, I_, X_);
        else if (N <= 8) e = run_barrier<double, 8>(*cfg, count, P_, N_, num_obstacles, O_, M_, C_, I_, X_);
        else e = run_barrier<double, 16>(*cfg, count, P_, N_, num_obstacles, O_, M_, C_, I_, X_);
    } else {
        if (N <= 4) e = run_barrier<float, 4>(*cfg, count, P_, N_, num_obstacles, O_, M_, C_, I_, X_);
        else if (N <= 8) e = run_barrier<float, 8>(*cfg, count, P_, N_, num_obstacles, O_, M_, C_, I_, X_);
        else e = run_barrier<float, 16>(*cfg, count, P_, N_, num_obstacles, O_, M_, C_, I_, X_);
    }
    if (e != cudaSuccess || cudaDeviceSynchronize() != cudaSuccess) return MRSIM_E_CUDA;
    std::vector<int32_t> co(count);
    cudaMemcpy(commands_out, C_, sizeof(double) * count * N * 2, cudaMemcpyDeviceToHost);
    cudaMemcpy(infeasible_out, I_, sizeof(int32_t) * count, cudaMemcpyDeviceToHost);
    cudaMemcpy(co.data(), X_, sizeof(int32_t) * count, cudaMemcpyDeviceToHost);
    for (int t = 0; t < count; ++t)
        if (co[t]) return MRSIM_E_DOMAIN;  // coincident robot positions (barrier.hpp:73-74)
    return MRSIM_OK;
}

}  // extern "C"
