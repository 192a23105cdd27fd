// policy.cuh — on-device feedforward policy, the producer of the step's
// actions (Policy::act with PolicyKind::FeedforwardFile, policy.hpp:445-480;
// FeedforwardWeights::forward, policy.hpp:95-116; harness.hpp:238-252).
//
// Teams of <= 4 robots: one warp per environment (lanes own (robot, neuron) outputs,
// four independent accumulation chains). Larger teams: a block owns a tile of
// consecutive environments (~32 robots): it stages
// their state in shared memory, assembles every robot's observation (the same
// features the step kernel stores, unrounded, in the state precision) as the
// rows of X [robots][inputs], and runs each dense layer as a small GEMM
// Y = act(b + X W^T) in which a thread owns a 4 x 4 register tile (4 robots x
// 4 neurons): per input it loads 4 activations (shared memory, broadcast
// across the warp) and 4 weights (transposed [in][out], coalesced through
// L1) for 16 multiply-adds. Thread r then picks robot r's action: greedy
// argmax (strict `>`, first maximum wins) or a softmax sample from
// policy_stream(episode seed, step, robot).
//
// Arithmetic: each neuron is b + w0*x0 + w1*x1 + ... accumulated in input
// order with explicitly rounded multiply and add (no FMA contraction), the
// reference's loop exactly; relu/identity layers are therefore bit-exact
// against the reference, tanh and the softmax exp differ by <= 1 ulp
// (device libm vs glibc), which can only flip near-tied decisions.
#pragma once

#include "step_kernel.cuh"

namespace mrsim_dev {

constexpr int kPolicyMaxLayers = 8;
constexpr int kPolicyMaxWidth = 256;
constexpr int kPolicyWarps = 4;  // warps per block (scripted planner)
constexpr int kPolicyTileThreads = 128;   // feedforward policy: threads per tile block
constexpr int kPolicyTileRobots = 32;     // robots per tile (whole envs)
constexpr int kPolicyTileSmem = 112 * 1024;  // shared-memory budget per tile block

struct PolicyNet {
    int num_layers;
    int in[kPolicyMaxLayers], out[kPolicyMaxLayers], act[kPolicyMaxLayers];  // act: MRSIM_ACT_*
    long long w_off[kPolicyMaxLayers], b_off[kPolicyMaxLayers];             // into wT / bias
    int greedy;
};

template <class Real>
struct PolicyParams {
    mrsim_cfg c;
    DevState<Real> s;
    long long B;
    int N, D, bdim, nf, ni;
    int maxw;          // max(D, layer widths): row stride of the activation buffers
    int tile_envs;     // tile kernel: envs per block (kPolicyTileRobots / N, fewer for wide layers)
    int warp_bytes;    // warp kernel: dynamic shared memory per warp
    const double* wT;  // per layer [in][out]
    const double* bias;
    PolicyNet net;
    int num_sms;       // of the context's device (grid sizing)
    int8_t* actions;   // [B][N]
};

// Per-env state staging in the tile's shared memory.
template <class Real>
struct PolicyStage {
    Real xs[MRSIM_MAX_ROBOTS], ys[MRSIM_MAX_ROBOTS], ts[MRSIM_MAX_ROBOTS], tf[kTfMax];
    int ti[kTiMax];
    int drones[MRSIM_MAX_ROBOTS];
};
template <class Real>
__host__ __device__ constexpr int policy_stage_bytes() {
    return (static_cast<int>(sizeof(PolicyStage<Real>)) + 15) & ~15;
}
// Shared memory of a tile of `envs` envs: staging, then two activation buffers [rows][maxw]
// (rows rounded up to the 4-robot register tiles).
template <class Real>
__host__ __device__ constexpr int policy_tile_bytes(int envs, int N, int maxw) {
    return envs * policy_stage_bytes<Real>() + 2 * (((envs * N + 3) / 4) * 4) * maxw * 8;
}
// Envs per tile: whole envs, about kPolicyTileRobots robots, within the shared-memory budget.
template <class Real>
__host__ __device__ inline int policy_tile_envs(int N, int maxw) {
    int envs = kPolicyTileRobots / N > 0 ? kPolicyTileRobots / N : 1;
    while (envs > 1 && policy_tile_bytes<Real>(envs, N, maxw) > kPolicyTileSmem) --envs;
    return envs;
}

// Warp kernel (small teams): per-warp shared memory, state staging then two activation buffers [N][maxw].
template <class Real>
__host__ __device__ constexpr int policy_warp_bytes(int N, int maxw) {
    return policy_stage_bytes<Real>() + 2 * N * maxw * 8;
}

// Small teams (N <= kPolicyWarpMaxN): one warp per env, lanes own (robot, neuron) outputs with four
// independent accumulation chains (round 1's kernel). Larger teams: the tiled GEMM below.
// Measured crossover (profiles/r02/ab_policy_tiles.log, policy + step): navigation N=4 0.721 vs
// 0.823 ms (warp), discovery N=6 1.344 vs 1.257 ms and MT N=10 12.70 vs 11.77 ms (tile).
constexpr int kPolicyWarpMaxN = 4;

template <class Real, int TASK>
__global__ void __launch_bounds__(32 * kPolicyWarps) policy_warp_kernel(const __grid_constant__ PolicyParams<Real> p) {
    extern __shared__ __align__(16) unsigned char pol_smem[];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    unsigned char* base = pol_smem + wib * p.warp_bytes;
    PolicyStage<Real>& sm = *reinterpret_cast<PolicyStage<Real>*>(base);
    double* bufs = reinterpret_cast<double*>(base + ((static_cast<int>(sizeof(PolicyStage<Real>)) + 15) & ~15));
    const mrsim_cfg& c = p.c;
    const int N = p.N, W = p.maxw;
    if (lane == 0) arctic_drones(c, sm.drones);
    const EnvView<Real> view{sm.xs, sm.ys, sm.ts, sm.tf, sm.ti, N, sm.drones, nullptr};
    const long long stride = static_cast<long long>(gridDim.x) * (blockDim.x >> 5);
    for (long long e = static_cast<long long>(blockIdx.x) * (blockDim.x >> 5) + wib; e < p.B; e += stride) {
        __syncwarp();
        if (lane < N) {
            sm.xs[lane] = p.s.px[e * N + lane];
            sm.ys[lane] = p.s.py[e * N + lane];
            sm.ts[lane] = p.s.pt[e * N + lane];
        }
        for (int f = lane; f < p.nf; f += 32) sm.tf[f] = p.s.tf[static_cast<long long>(f) * p.B + e];
        for (int w = lane; w < p.ni; w += 32) sm.ti[w] = p.s.ti[static_cast<long long>(w) * p.B + e];
        const int step = p.s.step_index[e];
        const uint64_t pkey = p.s.pkey[e];
        __syncwarp();
        // every robot's observation (assemble_observations, batch.hpp:143-151), unrounded
        double* x = bufs;
        double* y = bufs + N * W;
        for (int q = lane; q < N * p.D; q += 32) {
            const int r = q / p.D, f = q - r * p.D;
            x[r * W + f] = double(obs_feature<TASK, Real>(c, view, r, f, p.bdim));
        }
        __syncwarp();
        // FeedforwardWeights::forward (policy.hpp:95-116) for all robots at once: a lane owns
        // (robot, neuron) outputs and runs up to four of them as independent accumulation chains
        for (int l = 0; l < p.net.num_layers; ++l) {
            const int nin = p.net.in[l], nout = p.net.out[l], act = p.net.act[l];
            const double* Wt = p.wT + p.net.w_off[l];
            const double* bb = p.bias + p.net.b_off[l];
            const int total = N * nout;
            for (int b0 = lane; b0 < total; b0 += 128) {
                int ro[4], oo[4];
                double acc[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int idx = b0 + 32 * u;
                    const int idc = idx < total ? idx : b0;
                    ro[u] = idc / nout;
                    oo[u] = idc - ro[u] * nout;
                    acc[u] = __ldg(bb + oo[u]);
                }
                // chains live in this pass (warp-uniform): a small last layer (nav: 4 robots x 5
                // actions = 20 outputs) needs one, not four
                const int live = total - (b0 - lane);
                if (live > 96 && nout == 32) {
                    // chain u is robot 4k+u, neuron `lane`: one weight serves all four chains
                    for (int i = 0; i < nin; ++i) {
                        const double w = __ldg(Wt + static_cast<long long>(i) * 32 + lane);
#pragma unroll
                        for (int u = 0; u < 4; ++u) acc[u] = __dadd_rn(acc[u], __dmul_rn(w, x[ro[u] * W + i]));
                    }
                } else if (live > 96) {
                    for (int i = 0; i < nin; ++i) {
                        const double* wrow = Wt + static_cast<long long>(i) * nout;
#pragma unroll
                        for (int u = 0; u < 4; ++u)
                            acc[u] = __dadd_rn(acc[u], __dmul_rn(__ldg(wrow + oo[u]), x[ro[u] * W + i]));
                    }
                } else {
                    for (int i = 0; i < nin; ++i) {
                        const double* wrow = Wt + static_cast<long long>(i) * nout;
#pragma unroll
                        for (int u = 0; u < 4; ++u)
                            if (32 * u < live)
                                acc[u] = __dadd_rn(acc[u], __dmul_rn(__ldg(wrow + oo[u]), x[ro[u] * W + i]));
                    }
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    double v = acc[u];
                    if (act == MRSIM_ACT_RELU) v = v > 0 ? v : 0.0;
                    else if (act == MRSIM_ACT_TANH) v = tanh(v);
                    if (b0 + 32 * u < total) y[ro[u] * W + oo[u]] = v;
                }
            }
            __syncwarp();
            double* t = x;
            x = y;
            y = t;
        }
        if (lane < N) {  // Policy::act (policy.hpp:456-480), lane r for robot r
            const double* lg = x + lane * W;
            int a = 0;
            if (p.net.greedy) {
                for (int k = 1; k < 5; ++k)
                    if (lg[k] > lg[a]) a = k;
            } else {
                double mx = lg[0];
                for (int k = 0; k < 5; ++k) mx = mx < lg[k] ? lg[k] : mx;  // std::max
                double pr[5], z = 0.0;
                for (int k = 0; k < 5; ++k) {
                    pr[k] = exp(__dsub_rn(lg[k], mx));
                    z = __dadd_rn(z, pr[k]);
                }
                Rng rng{fork_key(fork_key(pkey, static_cast<uint64_t>(step)), static_cast<uint64_t>(lane)), 0};
                double u = __dmul_rn(rng.uniform(), z);
                a = 4;
                for (int k = 0; k < 5; ++k) {
                    u = __dsub_rn(u, pr[k]);
                    if (u <= 0.0) {
                        a = k;
                        break;
                    }
                }
            }
            p.actions[e * N + lane] = static_cast<int8_t>(a);
        }
    }
}

template <class Real, int TASK>
__global__ void __launch_bounds__(kPolicyTileThreads) policy_tile_kernel(const __grid_constant__ PolicyParams<Real> p) {
    extern __shared__ __align__(16) unsigned char pol_smem[];
    const mrsim_cfg& c = p.c;
    const int N = p.N, W = p.maxw, D = p.D;
    const long long e0 = static_cast<long long>(blockIdx.x) * p.tile_envs;
    const int ne = static_cast<int>(p.B - e0 < p.tile_envs ? p.B - e0 : p.tile_envs);
    const int R = ne * N;                         // robots of this tile
    const int RP = ((p.tile_envs * N + 3) / 4) * 4;  // rows of the activation buffers
    PolicyStage<Real>* st = reinterpret_cast<PolicyStage<Real>*>(pol_smem);
    double* X = reinterpret_cast<double*>(pol_smem + p.tile_envs * policy_stage_bytes<Real>());
    double* Y = X + RP * W;
    // ---- stage the tile's envs (coalesced: consecutive threads, consecutive envs) ----
    for (int k = threadIdx.x; k < R; k += blockDim.x) {
        const int le = k / N, r = k - le * N;
        const long long g = (e0 + le) * N + r;
        st[le].xs[r] = p.s.px[g];
        st[le].ys[r] = p.s.py[g];
        st[le].ts[r] = p.s.pt[g];
    }
    for (int k = threadIdx.x; k < ne * p.nf; k += blockDim.x) {
        const int f = k / ne, le = k - f * ne;
        st[le].tf[f] = p.s.tf[static_cast<long long>(f) * p.B + e0 + le];
    }
    for (int k = threadIdx.x; k < ne * p.ni; k += blockDim.x) {
        const int w = k / ne, le = k - w * ne;
        st[le].ti[w] = p.s.ti[static_cast<long long>(w) * p.B + e0 + le];
    }
    if (threadIdx.x < ne) arctic_drones(c, st[threadIdx.x].drones);
    __syncthreads();
    // ---- every robot's observation (assemble_observations, batch.hpp:143-151), unrounded ----
    for (int k = threadIdx.x; k < R * D; k += blockDim.x) {
        const int rr = k / D, f = k - rr * D;
        const int le = rr / N, r = rr - le * N;
        const EnvView<Real> view{st[le].xs, st[le].ys, st[le].ts, st[le].tf, st[le].ti, N, st[le].drones, nullptr};
        X[rr * W + f] = double(obs_feature<TASK, Real>(c, view, r, f, p.bdim));
    }
    __syncthreads();
    // ---- FeedforwardWeights::forward (policy.hpp:95-116): one small GEMM per layer ----
    for (int l = 0; l < p.net.num_layers; ++l) {
        const int nin = p.net.in[l], nout = p.net.out[l], act = p.net.act[l];
        const double* Wt = p.wT + p.net.w_off[l];
        const double* bb = p.bias + p.net.b_off[l];
        const int tr = (R + 3) / 4, tc = (nout + 3) / 4;
        for (int t = threadIdx.x; t < tr * tc; t += blockDim.x) {
            const int r0 = (t / tc) * 4, o0 = (t - (t / tc) * tc) * 4;
            double acc[4][4];
#pragma unroll
            for (int v = 0; v < 4; ++v) {
                const double b = (o0 + v < nout) ? __ldg(bb + o0 + v) : 0.0;
#pragma unroll
                for (int u = 0; u < 4; ++u) acc[u][v] = b;
            }
            const double* xr = X + r0 * W;
            for (int i = 0; i < nin; ++i) {
                double w[4], xv[4];
                const double* wrow = Wt + static_cast<long long>(i) * nout + o0;
#pragma unroll
                for (int v = 0; v < 4; ++v) w[v] = (o0 + v < nout) ? __ldg(wrow + v) : 0.0;
#pragma unroll
                for (int u = 0; u < 4; ++u) xv[u] = xr[u * W + i];
#pragma unroll
                for (int u = 0; u < 4; ++u)
#pragma unroll
                    for (int v = 0; v < 4; ++v) acc[u][v] = __dadd_rn(acc[u][v], __dmul_rn(w[v], xv[u]));
            }
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
                for (int v = 0; v < 4; ++v) {
                    if (r0 + u < R && o0 + v < nout) {
                        double a = acc[u][v];
                        if (act == MRSIM_ACT_RELU) a = a > 0 ? a : 0.0;
                        else if (act == MRSIM_ACT_TANH) a = tanh(a);
                        Y[(r0 + u) * W + o0 + v] = a;
                    }
                }
        }
        __syncthreads();
        double* tmp = X;
        X = Y;
        Y = tmp;
    }
    // ---- Policy::act (policy.hpp:456-480): one thread per robot ----
    for (int k = threadIdx.x; k < R; k += blockDim.x) {
        const int le = k / N, r = k - le * N;
        const long long e = e0 + le;
        const double* lg = X + k * W;
        int a = 0;
        if (p.net.greedy) {
            for (int q = 1; q < 5; ++q)
                if (lg[q] > lg[a]) a = q;
        } else {
            double mx = lg[0];
            for (int q = 0; q < 5; ++q) mx = mx < lg[q] ? lg[q] : mx;  // std::max
            double pr[5], z = 0.0;
            for (int q = 0; q < 5; ++q) {
                pr[q] = exp(__dsub_rn(lg[q], mx));
                z = __dadd_rn(z, pr[q]);
            }
            Rng rng{fork_key(fork_key(p.s.pkey[e], static_cast<uint64_t>(p.s.step_index[e])), static_cast<uint64_t>(r)),
                    0};
            double u = __dmul_rn(rng.uniform(), z);
            a = 4;
            for (int q = 0; q < 5; ++q) {
                u = __dsub_rn(u, pr[q]);
                if (u <= 0.0) {
                    a = q;
                    break;
                }
            }
        }
        p.actions[e * N + r] = static_cast<int8_t>(a);
    }
}

}  // namespace mrsim_dev
