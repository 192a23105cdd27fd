// policy.cuh — on-device feedforward policy, the producer of the step's
// actions (Policy::act with PolicyKind::FeedforwardFile, policy.hpp:445-480;
// FeedforwardWeights::forward, policy.hpp:95-116; harness.hpp:238-252).
//
// One warp per environment. The warp stages the env's state in shared
// memory, then per robot: assembles the observation (the same features the
// step kernel stores, unrounded, in the state precision), runs the dense
// layers with lanes splitting the output neurons (weights stored transposed
// [in][out] so a warp's loads of one input row are contiguous), and lane 0
// picks the action: greedy argmax (strict `>`, first maximum wins) or a
// softmax sample from policy_stream(episode seed, step, robot).
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
constexpr int kPolicyWarps = 4;  // warps per block

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
    const double* wT;  // per layer [in][out]
    const double* bias;
    PolicyNet net;
    int8_t* actions;   // [B][N]
};

// Per-warp shared memory: state staging + two activation buffers.
template <class Real>
struct PolicySmem {
    Real xs[MRSIM_MAX_ROBOTS], ys[MRSIM_MAX_ROBOTS], ts[MRSIM_MAX_ROBOTS], tf[kTfMax];
    int ti[kTiMax];
    int drones[MRSIM_MAX_ROBOTS];
    double h[2][kPolicyMaxWidth];
};

template <class Real, int TASK>
__global__ void __launch_bounds__(32 * kPolicyWarps) policy_kernel(const __grid_constant__ PolicyParams<Real> p) {
    __shared__ PolicySmem<Real> smem[kPolicyWarps];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    PolicySmem<Real>& sm = smem[wib];
    const mrsim_cfg& c = p.c;
    const int N = p.N;
    if (lane == 0) arctic_drones(c, sm.drones);
    const EnvView<Real> view{sm.xs, sm.ys, sm.ts, sm.tf, sm.ti, N, sm.drones, nullptr};
    const long long stride = static_cast<long long>(gridDim.x) * kPolicyWarps;
    for (long long e = static_cast<long long>(blockIdx.x) * kPolicyWarps + wib; e < p.B; e += stride) {
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
        for (int r = 0; r < N; ++r) {
            // observation of robot r (assemble_observations, batch.hpp:143-151)
            for (int q = lane; q < p.D; q += 32) sm.h[0][q] = double(obs_feature<TASK, Real>(c, view, r, q, p.bdim));
            __syncwarp();
            int cur = 0;
            for (int l = 0; l < p.net.num_layers; ++l) {  // FeedforwardWeights::forward (policy.hpp:95-116)
                const int nin = p.net.in[l], nout = p.net.out[l], act = p.net.act[l];
                const double* W = p.wT + p.net.w_off[l];
                const double* bb = p.bias + p.net.b_off[l];
                const double* x = sm.h[cur];
                double* y = sm.h[cur ^ 1];
                for (int o = lane; o < nout; o += 32) {
                    double acc = __ldg(bb + o);
                    for (int i = 0; i < nin; ++i) acc = __dadd_rn(acc, __dmul_rn(__ldg(W + static_cast<long long>(i) * nout + o), x[i]));
                    if (act == MRSIM_ACT_RELU) acc = acc > 0 ? acc : 0.0;
                    else if (act == MRSIM_ACT_TANH) acc = tanh(acc);
                    y[o] = acc;
                }
                __syncwarp();
                cur ^= 1;
            }
            if (lane == 0) {  // Policy::act (policy.hpp:456-480)
                const double* lg = sm.h[cur];
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
                    Rng rng{fork_key(fork_key(pkey, static_cast<uint64_t>(step)), static_cast<uint64_t>(r)), 0};
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
                p.actions[e * N + r] = static_cast<int8_t>(a);
            }
            __syncwarp();
        }
    }
}

}  // namespace mrsim_dev
