// capi.cu — the C ABI of include/mrsim_cuda.h: context lifetime, batch
// state in HBM (two ping-pong SoA copies), kernel dispatch per
// (task, group width, precision), host-buffer step, state/stats I/O and
// device error reporting. No CPU fallback exists: every compute entry point
// launches the sm_100a kernels or fails with MRSIM_E_CUDA.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <algorithm>
#include <string>
#include <thread>
#include <vector>

#include "launch.h"
#include "mrsim_cuda.h"

using mrsim_dev::DevState;
using mrsim_dev::EnvStats;
using mrsim_dev::ResetParams;
using mrsim_dev::StepParams;

// Warp-staged obs stores on the device-buffer path too (not only for zero-copy host buffers):
// measured -3.7 % nav N=4, neutral elsewhere (profiles/r02/ab_obs_stage.log), so off.
#ifndef MRSIM_STAGE_DEVICE_OBS
#define MRSIM_STAGE_DEVICE_OBS 0
#endif

struct mrsim_ctx {
    mrsim_cfg cfg;
    int device = 0;
    long long B = 0;
    unsigned flags = 0;
    bool fp64 = false;
    int N = 0, n = 0, P = 0, D = 0, bdim = 0, nf = 0, ni = 0, L = 8;
    mrsim_host::Variant var{4, 2, 0};
    void* mem[2] = {nullptr, nullptr};
    DevState<float> sf[2];
    DevState<double> sd[2];
    void* stats_mem = nullptr;
    EnvStats st{};
    unsigned long long* d_err = nullptr;
    long long* d_err_serial = nullptr;
    unsigned* d_ticket = nullptr;
    unsigned* d_exit = nullptr;  // step kernel's finished-warp counter (err_epilogue)
    long long scripted_launches = 0;
    int cur = 0;
    long long serial = 0;
    bool has_episodes = false;
    uint64_t root_seed = 0;
    long long episode_stride = 0;
    long long env_steps = 0;
    std::string last_error;
    std::vector<std::pair<char*, size_t>> guard_tails;  // checks builds: allocation guard tails
    int num_sms = 148;
    int block = 128;
    int grid = 0;
    int grid_staged = 0;  // the grid of launches with the warp obs stage (host-buffer steps)
    int smem_group = 0;
    int obs_stage = 0;  // floats per warp of the staged obs store (0: direct stores)
    bool obs_ws_ok = false;  // an env's obs fit its group's QP inverse-Gram matrix (the fallback stage)
    // host-API scratch
    float* d_obs = nullptr;
    double* d_reward64 = nullptr;
    uint8_t* d_done = nullptr;
    unsigned long long* h_err = nullptr;  // pinned copy of the device error word + serial
    void* h_state = nullptr;              // pinned host mirror of one state copy (state I/O)
    int32_t* d_actions32 = nullptr;
    bool reset_done = false;
    // on-device policy: feedforward network (mrsim_set_policy_feedforward) or scripted (kind != 0)
    int scripted = 0;
    bool ff = false;
    mrsim_dev::PolicyNet net{};
    double* d_wT = nullptr;
    double* d_bias = nullptr;
    int8_t* d_pol_actions = nullptr;
    // trajectory capture (mrsim_capture_begin)
    mrsim_traj_record* d_cap = nullptr;
    long long cap_max = 0, cap_steps = 0;
};

namespace mrsim_dev {
__global__ void stats_rollback_kernel(EnvStats st, long long serial, long long B) {
    const long long e = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (e >= B || st.upd_serial[e] != serial) return;
    st.episodes[e] = st.u_episodes[e];
    st.ret[e] = st.u_ret[e];
    st.ret_sq[e] = st.u_ret_sq[e];
    st.metric[e] = st.u_metric[e];
    st.success[e] = st.u_success[e];
    st.min_dist[e] = st.u_min_dist[e];
    st.collisions[e] = st.u_collisions[e];
    st.qp_inf[e] = st.u_qp_inf[e];
    st.upd_serial[e] = -1;
}
}  // namespace mrsim_dev

namespace {

int set_err(mrsim_ctx* ctx, int code, const std::string& msg) {
    if (ctx) ctx->last_error = msg;
    return code;
}

int cuda_fail(mrsim_ctx* ctx, cudaError_t e, const char* where) {
    return set_err(ctx, MRSIM_E_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

#define CK(expr)                                                    \
    do {                                                            \
        cudaError_t _e = (expr);                                    \
        if (_e != cudaSuccess) return cuda_fail(ctx, _e, #expr);    \
    } while (0)

// SoA state copy layout: the fields in carve order, each 256-byte aligned (plus a guard gap
// behind every field in -DMRSIM_DEVICE_CHECKS builds, verified by mrsim_debug_check_guards).
#ifdef MRSIM_DEVICE_CHECKS
constexpr size_t kStateGuard = 256;
constexpr size_t kAllocGuard = 256;
#else
constexpr size_t kStateGuard = 0;
constexpr size_t kAllocGuard = 0;
#endif
constexpr int kStateFields = 16;

template <class Real>
void state_field_bytes(long long B, int N, int nf, int ni, size_t (&f)[kStateFields]) {
    const size_t R = sizeof(Real);
    const size_t v[kStateFields] = {R * B * N, R * B * N, R * B * N,            // px, py, pt
                                    4 * size_t(B),                              // step_index
                                    8 * size_t(B), 8 * size_t(B), 8 * size_t(B),  // key, seed, pkey
                                    8 * size_t(B),                              // episode
                                    4 * size_t(B), 4 * size_t(B), 4 * size_t(B),  // collisions, qp_inf, success
                                    R * B, R * B, R * B,                        // metric, min_dist, ep_return
                                    R * B * (nf > 0 ? nf : 1), 4 * size_t(B) * (ni > 0 ? ni : 1)};  // tf, ti
    for (int k = 0; k < kStateFields; ++k) f[k] = v[k];
}
inline size_t state_slot(size_t bytes) { return ((bytes + 255) & ~size_t(255)) + kStateGuard; }

template <class Real>
size_t state_bytes(long long B, int N, int nf, int ni) {
    size_t f[kStateFields], b = 0;
    state_field_bytes<Real>(B, N, nf, ni, f);
    for (size_t x : f) b += state_slot(x);
    return b;
}

template <class Real>
void carve_state(void* base, long long B, int N, int nf, int ni, DevState<Real>& s) {
    size_t f[kStateFields];
    state_field_bytes<Real>(B, N, nf, ni, f);
    char* p = static_cast<char*>(base);
    char* at[kStateFields];
    for (int k = 0; k < kStateFields; ++k) {
        at[k] = p;
        p += state_slot(f[k]);
    }
    s.px = reinterpret_cast<Real*>(at[0]);
    s.py = reinterpret_cast<Real*>(at[1]);
    s.pt = reinterpret_cast<Real*>(at[2]);
    s.step_index = reinterpret_cast<int32_t*>(at[3]);
    s.key = reinterpret_cast<uint64_t*>(at[4]);
    s.seed = reinterpret_cast<uint64_t*>(at[5]);
    s.pkey = reinterpret_cast<uint64_t*>(at[6]);
    s.episode = reinterpret_cast<int64_t*>(at[7]);
    s.collisions = reinterpret_cast<int32_t*>(at[8]);
    s.qp_inf = reinterpret_cast<int32_t*>(at[9]);
    s.success = reinterpret_cast<int32_t*>(at[10]);
    s.metric = reinterpret_cast<Real*>(at[11]);
    s.min_dist = reinterpret_cast<Real*>(at[12]);
    s.ep_return = reinterpret_cast<Real*>(at[13]);
    s.tf = reinterpret_cast<Real*>(at[14]);
    s.ti = reinterpret_cast<int32_t*>(at[15]);
}

// Guard regions of a state copy at `base`: [offset, offset + kStateGuard) behind every field.
template <class Real>
void state_guards(long long B, int N, int nf, int ni, std::vector<size_t>& offsets) {
    size_t f[kStateFields], b = 0;
    state_field_bytes<Real>(B, N, nf, ni, f);
    for (size_t x : f) {
        b += state_slot(x);
        offsets.push_back(b - kStateGuard);
    }
}

// Device allocation owned by the context: in checks builds with a guard tail of kAllocGuard
// pattern bytes, registered for mrsim_debug_check_guards.
template <class T>
cudaError_t ctx_malloc(mrsim_ctx* ctx, T** ptr, size_t bytes) {
    cudaError_t e = cudaMalloc(reinterpret_cast<void**>(ptr), bytes + kAllocGuard);
    if (e != cudaSuccess || !kAllocGuard) return e;
    e = cudaMemset(reinterpret_cast<char*>(*ptr) + bytes, 0xA5, kAllocGuard);
    ctx->guard_tails.emplace_back(reinterpret_cast<char*>(*ptr) + bytes, kAllocGuard);
    return e;
}
// cudaFree of a ctx_malloc allocation, dropping its guard tail: the registered tail nearest
// above the allocation's start (allocations do not overlap).
template <class T>
void ctx_free(mrsim_ctx* ctx, T* ptr) {
    if (!ptr) return;
    if (kAllocGuard) {
        char* const lo = reinterpret_cast<char*>(ptr);
        size_t best = ctx->guard_tails.size();
        for (size_t i = 0; i < ctx->guard_tails.size(); ++i)
            if (ctx->guard_tails[i].first >= lo &&
                (best == ctx->guard_tails.size() || ctx->guard_tails[i].first < ctx->guard_tails[best].first))
                best = i;
        if (best < ctx->guard_tails.size()) ctx->guard_tails.erase(ctx->guard_tails.begin() + best);
    }
    cudaFree(ptr);
}

// ---- dispatch tables over the task template parameter ----
template <class Real>
cudaError_t dispatch_step(int task, const StepParams<Real>& p, mrsim_host::Variant v, int grid, int block, int smem,
                          cudaStream_t s) {
    using namespace mrsim_host;
    switch (task) {
        case 0: return launch_step<Real, 0>(p, v, grid, block, smem, s);
        case 1: return launch_step<Real, 1>(p, v, grid, block, smem, s);
        case 2: return launch_step<Real, 2>(p, v, grid, block, smem, s);
        case 3: return launch_step<Real, 3>(p, v, grid, block, smem, s);
        case 4: return launch_step<Real, 4>(p, v, grid, block, smem, s);
        case 5: return launch_step<Real, 5>(p, v, grid, block, smem, s);
        case 6: return launch_step<Real, 6>(p, v, grid, block, smem, s);
        case 7: return launch_step<Real, 7>(p, v, grid, block, smem, s);
        default: return launch_step<Real, 8>(p, v, grid, block, smem, s);
    }
}
template <class Real>
cudaError_t dispatch_occ(int task, mrsim_host::Variant v, int block, int smem, int* bps) {
    using namespace mrsim_host;
    switch (task) {
        case 0: return step_occupancy<Real, 0>(v, block, smem, bps);
        case 1: return step_occupancy<Real, 1>(v, block, smem, bps);
        case 2: return step_occupancy<Real, 2>(v, block, smem, bps);
        case 3: return step_occupancy<Real, 3>(v, block, smem, bps);
        case 4: return step_occupancy<Real, 4>(v, block, smem, bps);
        case 5: return step_occupancy<Real, 5>(v, block, smem, bps);
        case 6: return step_occupancy<Real, 6>(v, block, smem, bps);
        case 7: return step_occupancy<Real, 7>(v, block, smem, bps);
        default: return step_occupancy<Real, 8>(v, block, smem, bps);
    }
}
template <class Real>
cudaError_t dispatch_reset(int task, const ResetParams<Real>& p, cudaStream_t s) {
    using namespace mrsim_host;
    switch (task) {
        case 0: return launch_reset<Real, 0>(p, s);
        case 1: return launch_reset<Real, 1>(p, s);
        case 2: return launch_reset<Real, 2>(p, s);
        case 3: return launch_reset<Real, 3>(p, s);
        case 4: return launch_reset<Real, 4>(p, s);
        case 5: return launch_reset<Real, 5>(p, s);
        case 6: return launch_reset<Real, 6>(p, s);
        case 7: return launch_reset<Real, 7>(p, s);
        default: return launch_reset<Real, 8>(p, s);
    }
}

template <class Real>
cudaError_t dispatch_policy(int task, const mrsim_dev::PolicyParams<Real>& p, cudaStream_t s) {
    using namespace mrsim_host;
    switch (task) {
        case 0: return launch_policy<Real, 0>(p, s);
        case 1: return launch_policy<Real, 1>(p, s);
        case 2: return launch_policy<Real, 2>(p, s);
        case 3: return launch_policy<Real, 3>(p, s);
        case 4: return launch_policy<Real, 4>(p, s);
        case 5: return launch_policy<Real, 5>(p, s);
        case 6: return launch_policy<Real, 6>(p, s);
        case 7: return launch_policy<Real, 7>(p, s);
        default: return launch_policy<Real, 8>(p, s);
    }
}

template <class Real>
cudaError_t dispatch_scripted(int task, const mrsim_dev::ScriptedParams<Real>& p, cudaStream_t s) {
    using namespace mrsim_host;
    switch (task) {
        case 0: return launch_scripted<Real, 0>(p, s);
        case 1: return launch_scripted<Real, 1>(p, s);
        case 2: return launch_scripted<Real, 2>(p, s);
        case 3: return launch_scripted<Real, 3>(p, s);
        case 4: return launch_scripted<Real, 4>(p, s);
        case 5: return launch_scripted<Real, 5>(p, s);
        case 6: return launch_scripted<Real, 6>(p, s);
        case 7: return launch_scripted<Real, 7>(p, s);
        default: return launch_scripted<Real, 8>(p, s);
    }
}

template <class Real>
cudaError_t scripted_launch(mrsim_ctx* ctx, const DevState<Real>& st, int8_t* out, cudaStream_t s) {
    mrsim_dev::ScriptedParams<Real> p;
    std::memset(&p, 0, sizeof p);
    p.c = ctx->cfg;
    p.s = st;
    p.B = ctx->B;
    p.N = ctx->N;
    p.nf = ctx->nf;
    p.ni = ctx->ni;
    p.kind = ctx->scripted;
    mrsim_dev::prey_offsets(ctx->cfg, p.prey_off);
    p.actions = out;
    p.ticket = ctx->d_ticket + 2;
    p.serial = ctx->scripted_launches;
    p.num_sms = ctx->num_sms;
    const cudaError_t e = dispatch_scripted<Real>(ctx->cfg.task, p, s);
    if (e == cudaSuccess) ++ctx->scripted_launches;  // the next launch clears the counter this one used
    return e;
}

template <class Real>
cudaError_t policy_launch(mrsim_ctx* ctx, const DevState<Real>& st, int8_t* out, cudaStream_t s) {
    if (ctx->scripted) return scripted_launch<Real>(ctx, st, out, s);
    mrsim_dev::PolicyParams<Real> p;
    p.c = ctx->cfg;
    p.s = st;
    p.B = ctx->B;
    p.N = ctx->N;
    p.D = ctx->D;
    p.bdim = ctx->bdim;
    p.nf = ctx->nf;
    p.ni = ctx->ni;
    p.wT = ctx->d_wT;
    p.bias = ctx->d_bias;
    p.net = ctx->net;
    int maxw = ctx->D;
    for (int l = 0; l < ctx->net.num_layers; ++l) maxw = maxw > ctx->net.out[l] ? maxw : ctx->net.out[l];
    p.maxw = maxw;
    p.tile_envs = 0;  // set by the launcher
    p.warp_bytes = 0;
    p.num_sms = ctx->num_sms;
    p.actions = out;
    return dispatch_policy<Real>(ctx->cfg.task, p, s);
}

template <class Real>
cudaError_t dispatch_observe(mrsim_ctx* ctx, const DevState<Real>& s, float* obs, cudaStream_t st) {
    using namespace mrsim_host;
    const mrsim_cfg& c = ctx->cfg;
    const int D = ctx->D, bd = ctx->bdim, nf = ctx->nf, ni = ctx->ni;
    const long long B = ctx->B;
    switch (c.task) {
        case 0: return launch_observe<Real, 0>(c, s, obs, B, D, bd, nf, ni, st);
        case 1: return launch_observe<Real, 1>(c, s, obs, B, D, bd, nf, ni, st);
        case 2: return launch_observe<Real, 2>(c, s, obs, B, D, bd, nf, ni, st);
        case 3: return launch_observe<Real, 3>(c, s, obs, B, D, bd, nf, ni, st);
        case 4: return launch_observe<Real, 4>(c, s, obs, B, D, bd, nf, ni, st);
        case 5: return launch_observe<Real, 5>(c, s, obs, B, D, bd, nf, ni, st);
        case 6: return launch_observe<Real, 6>(c, s, obs, B, D, bd, nf, ni, st);
        case 7: return launch_observe<Real, 7>(c, s, obs, B, D, bd, nf, ni, st);
        default: return launch_observe<Real, 8>(c, s, obs, B, D, bd, nf, ni, st);
    }
}

const char* err_text(unsigned code) {
    switch (code) {
        case mrsim_dev::kErrInvalidAction: return "step_batch: invalid action";
        case mrsim_dev::kErrCoincident: return "build_barrier_constraints: coincident robot positions";
        case mrsim_dev::kErrNonFinite: return "wrap_angle: non-finite input";
        case mrsim_dev::kErrSpawn: return "sample_poses: could not place robot";
        case mrsim_dev::kErrGoals: return "navigation: could not place goals";
        case mrsim_dev::kErrPrey: return "predator_prey: could not place prey";
        default: return "unknown device error";
    }
}
int err_code(unsigned code) {
    switch (code) {
        case mrsim_dev::kErrInvalidAction: return MRSIM_E_INVALID_ARGUMENT;
        case mrsim_dev::kErrCoincident:
        case mrsim_dev::kErrNonFinite: return MRSIM_E_DOMAIN;
        default: return MRSIM_E_RUNTIME;
    }
}

// Read the sticky device error word; returns MRSIM_OK or the mapped code.
int check_device_error(mrsim_ctx* ctx, bool rollback, const int32_t* host_actions = nullptr,
                       const unsigned long long* fetched = nullptr) {
    unsigned long long w = 0;
    long long ser = -1;
    if (fetched) {  // error word + serial already copied to host with the step's outputs
        w = fetched[0];
        if (w == ~0ull) return MRSIM_OK;
        ser = static_cast<long long>(fetched[1]);
    } else {
        cudaError_t e = cudaMemcpy(&w, ctx->d_err, sizeof w, cudaMemcpyDeviceToHost);
        if (e != cudaSuccess) return cuda_fail(ctx, e, "read device error");
        if (w == ~0ull) return MRSIM_OK;
        cudaMemcpy(&ser, ctx->d_err_serial, sizeof ser, cudaMemcpyDeviceToHost);
    }
    const unsigned code = static_cast<unsigned>(w & 0xff);
    const int detail = static_cast<int>((w >> 8) & 0xff);
    const int robot = static_cast<int>((w >> 16) & 0xff);
    const long long env = static_cast<long long>((w >> 24) & ((1ull << mrsim_dev::kErrEnvBits) - 1));
    char buf[256];
    if (code == mrsim_dev::kErrInvalidAction)  // the device keeps 8 bits; the host buffer has the full value
        std::snprintf(buf, sizeof buf, "step_batch: invalid action %d for environment %lld, robot %d",
                      host_actions ? host_actions[env * ctx->N + robot] : static_cast<int>(static_cast<int8_t>(detail)),
                      env, robot);
    else if (code == mrsim_dev::kErrSpawn)
        std::snprintf(buf, sizeof buf, "sample_poses: could not place robot %d after 1000 attempts (environment %lld)",
                      robot, env);
    else
        std::snprintf(buf, sizeof buf, "%s (environment %lld, robot %d)", err_text(code), env, robot);
    if (rollback && ser >= 0 && ser < ctx->serial) {
        // Every launched step flips the ping-pong index once and the steps after the failing
        // one are no-ops, so the failing step's (untouched) input buffer is the current one
        // flipped by the parity of the number of steps launched since.
        ctx->cur ^= static_cast<int>((ctx->serial - ser) & 1);
        const unsigned grid = static_cast<unsigned>((ctx->B + 255) / 256);
        mrsim_dev::stats_rollback_kernel<<<grid, 256>>>(ctx->st, ser, ctx->B);  // and its episode stats
        cudaDeviceSynchronize();
    }
    // clear so the context stays usable after the caller handled the error
    const unsigned long long none = ~0ull;
    cudaMemcpy(ctx->d_err, &none, sizeof none, cudaMemcpyHostToDevice);
    return set_err(ctx, err_code(code), buf);
}

template <class Real>
StepParams<Real> step_params(mrsim_ctx* ctx, DevState<Real>* s, const int8_t* actions, float* obs, float* reward,
                             uint8_t* done, float* next_obs, double* reward64, const int32_t* actions32) {
    StepParams<Real> p;
    std::memset(&p, 0, sizeof p);
    p.c = ctx->cfg;
    p.in = s[ctx->cur];
    p.out = s[1 - ctx->cur];
    p.st = ctx->st;
    p.actions = actions;
    p.actions32 = actions32;
    p.obs = obs;
    p.reward = reward;
    p.reward64 = reward64;
    p.done = done;
    p.next_obs = next_obs;
    p.err = ctx->d_err;
    p.err_serial = ctx->d_err_serial;
    p.ticket = ctx->d_ticket;
    p.serial = ctx->serial;
    p.exit_count = ctx->d_exit;
    p.err_host = nullptr;
    p.B = ctx->B;
    p.e_begin = 0;
    p.e_end = ctx->B;
    p.N = ctx->N;
    p.n = ctx->n;
    p.P = ctx->P;
    p.D = ctx->D;
    p.bdim = ctx->bdim;
    p.nf = ctx->nf;
    p.ni = ctx->ni;
    p.auto_reset = (ctx->flags & MRSIM_FLAG_AUTO_RESET) ? 1 : 0;
    p.n_steps = 1;
    p.obs_step_stride = static_cast<long long>(ctx->B) * ctx->N * ctx->D;
    p.root_seed = ctx->root_seed;
    p.episode_stride = ctx->episode_stride;
    p.smem_bytes_per_group = ctx->smem_group;
    p.obs_stage = ctx->obs_stage;
    mrsim_host::fill_consts(ctx->cfg, p.k);
    mrsim_dev::prey_offsets(ctx->cfg, p.prey_off);
    return p;
}

// Bookkeeping after every env of a step has been launched (ping-pong flip, rollback history).
void step_done(mrsim_ctx* ctx) {
    ctx->serial += 1;
    ctx->cur = 1 - ctx->cur;
    ctx->env_steps += ctx->B;
}

template <class Real>
int do_step(mrsim_ctx* ctx, DevState<Real>* s, const int8_t* actions, float* obs, float* reward, uint8_t* done,
            float* next_obs, cudaStream_t stream, double* reward64 = nullptr, const int32_t* actions32 = nullptr,
            bool stage_obs = false, unsigned long long* err_host = nullptr) {
    StepParams<Real> p = step_params<Real>(ctx, s, actions, obs, reward, done, next_obs, reward64, actions32);
    p.err_host = ctx->L > 1 ? err_host : nullptr;  // the env kernel has no epilogue: caller copies the word
    // warp-staged obs stores only where they pay: obs going straight to pinned host memory
    // (device-memory obs: ~2 % slower staged, measured)
    p.obs_stage = (stage_obs || ctx->L == 1 || MRSIM_STAGE_DEVICE_OBS) ? ctx->obs_stage : 0;
    p.obs_ws_stage = (stage_obs && ctx->L > 1 && !p.obs_stage && ctx->obs_ws_ok) ? 1 : 0;
    const int smem = ctx->smem_group * (ctx->block / ctx->L) + 4 * p.obs_stage * (ctx->block / 32);
    const int grid = (p.obs_stage && ctx->L > 1) ? ctx->grid_staged : ctx->grid;
    cudaError_t e = dispatch_step<Real>(ctx->cfg.task, p, ctx->var, grid, ctx->block, smem, stream);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "step kernel launch");
    step_done(ctx);
    return MRSIM_OK;
}

// Device-accessible alias of a host pointer: page-locked (pinned) host memory
// is mapped into the device address space, so the step kernel can read the
// actions and write obs / reward / done straight over the host link while it
// computes (no separate copy phase). nullptr for pageable memory.
template <class T>
T* mapped_alias(T* host) {
    if (!host) return nullptr;
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, host) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    if (a.type != cudaMemoryTypeHost || !a.devicePointer) return nullptr;
    return static_cast<T*>(a.devicePointer);
}

template <class Real>
int do_reset(mrsim_ctx* ctx, DevState<Real>* s, const uint64_t* d_seeds, uint64_t root, long long first,
             float* obs, cudaStream_t stream) {
    ResetParams<Real> p;
    std::memset(&p, 0, sizeof p);
    p.c = ctx->cfg;
    p.out = s[ctx->cur];
    p.seeds = d_seeds;
    p.root_seed = root;
    p.first_episode = first;
    p.obs = obs;
    p.err = ctx->d_err;
    p.B = ctx->B;
    p.N = ctx->N;
    p.D = ctx->D;
    p.bdim = ctx->bdim;
    p.nf = ctx->nf;
    p.ni = ctx->ni;
    cudaError_t e = dispatch_reset<Real>(ctx->cfg.task, p, stream);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "reset kernel launch");
    return MRSIM_OK;
}

// fn(k) for k in [0, count) on the host's cores (state conversions of large batches).
template <class F>
void host_parallel_for(long long count, F&& fn) {
    const long long T = static_cast<long long>(std::thread::hardware_concurrency());
    if (count < 8192 || T <= 1) {
        for (long long k = 0; k < count; ++k) fn(k);
        return;
    }
    const long long per = (count + T - 1) / T;
    std::vector<std::thread> pool;
    for (long long t = 0; t < T; ++t)
        pool.emplace_back([&, t] {
            const long long lo = t * per, hi = std::min(count, lo + per);
            for (long long k = lo; k < hi; ++k) fn(k);
        });
    for (auto& th : pool) th.join();
}

// Pinned host mirror of one state copy, carved exactly like the device copies.
template <class Real>
cudaError_t host_mirror(mrsim_ctx* ctx, DevState<Real>& h) {
    if (!ctx->h_state) {
        const cudaError_t e = cudaMallocHost(&ctx->h_state, state_bytes<Real>(ctx->B, ctx->N, ctx->nf, ctx->ni));
        if (e != cudaSuccess) {
            ctx->h_state = nullptr;
            return e;
        }
        if (kStateGuard) {  // whole-block uploads carry the mirror's guard gaps to the device copy
            std::vector<size_t> gaps;
            state_guards<Real>(ctx->B, ctx->N, ctx->nf, ctx->ni, gaps);
            for (size_t off : gaps) std::memset(static_cast<char*>(ctx->h_state) + off, 0xA5, kStateGuard);
        }
    }
    carve_state(ctx->h_state, ctx->B, ctx->N, ctx->nf, ctx->ni, h);
    return cudaSuccess;
}

// Copy envs [first, first + count) of every field between a device state copy and the host
// mirror: the whole block in one transfer for the full batch, else one slice per field.
template <class Real>
cudaError_t copy_state_slices(mrsim_ctx* ctx, const DevState<Real>& d, const DevState<Real>& h, long long first,
                              long long count, cudaMemcpyKind kind) {
    const bool up = kind == cudaMemcpyHostToDevice;
    if (first == 0 && count == ctx->B) {
        const size_t sb = state_bytes<Real>(ctx->B, ctx->N, ctx->nf, ctx->ni);
        return up ? cudaMemcpy(d.px, h.px, sb, kind) : cudaMemcpy(h.px, d.px, sb, kind);
    }
    cudaError_t e = cudaSuccess;
    auto cp = [&](void* dv, void* hv, size_t bytes) {
        if (e == cudaSuccess) e = up ? cudaMemcpy(dv, hv, bytes, kind) : cudaMemcpy(hv, dv, bytes, kind);
    };
    const int N = ctx->N;
    cp(d.px + first * N, h.px + first * N, sizeof(Real) * count * N);
    cp(d.py + first * N, h.py + first * N, sizeof(Real) * count * N);
    cp(d.pt + first * N, h.pt + first * N, sizeof(Real) * count * N);
    cp(d.step_index + first, h.step_index + first, 4 * count);
    cp(d.key + first, h.key + first, 8 * count);
    cp(d.seed + first, h.seed + first, 8 * count);
    cp(d.pkey + first, h.pkey + first, 8 * count);
    cp(d.episode + first, h.episode + first, 8 * count);
    cp(d.collisions + first, h.collisions + first, 4 * count);
    cp(d.qp_inf + first, h.qp_inf + first, 4 * count);
    cp(d.success + first, h.success + first, 4 * count);
    cp(d.metric + first, h.metric + first, sizeof(Real) * count);
    cp(d.min_dist + first, h.min_dist + first, sizeof(Real) * count);
    cp(d.ep_return + first, h.ep_return + first, sizeof(Real) * count);
    for (int f = 0; f < ctx->nf; ++f) cp(d.tf + f * ctx->B + first, h.tf + f * ctx->B + first, sizeof(Real) * count);
    for (int w = 0; w < ctx->ni; ++w) cp(d.ti + w * ctx->B + first, h.ti + w * ctx->B + first, 4 * count);
    return e;
}

template <class Real>
void to_host_states(mrsim_ctx* ctx, const DevState<Real>& s, long long first, long long count,
                    mrsim_env_state* out, cudaError_t* err) {
    const int N = ctx->N;
    // the device SoA block (or the requested env slice of each field) into its pinned host mirror
    DevState<Real> h;
    cudaError_t e = host_mirror<Real>(ctx, h);
    if (e == cudaSuccess) e = copy_state_slices<Real>(ctx, s, h, first, count, cudaMemcpyDeviceToHost);
    const Real *px = h.px + first * N, *py = h.py + first * N, *pt = h.pt + first * N;
    const Real *metric = h.metric + first, *mind = h.min_dist + first, *ret = h.ep_return + first;
    const int32_t *step = h.step_index + first, *coll = h.collisions + first, *qpi = h.qp_inf + first,
                  *succ = h.success + first;
    const uint64_t *key = h.key + first, *seed = h.seed + first;
    const int64_t* ep = h.episode + first;
    const Real* tf = h.tf + first;
    const int32_t* ti = h.ti + first;
    *err = e;
    if (e != cudaSuccess) return;
    const mrsim_cfg& c = ctx->cfg;
    const mrsim_layout& y = c.layout;
    host_parallel_for(count, [&](long long k) {
        mrsim_env_state& o = out[k];
        std::memset(&o, 0, sizeof o);
        o.num_robots = N;
        o.step_index = step[k];
        o.rng_key = key[k];
        o.seed = seed[k];
        o.episode = ep[k];
        for (int i = 0; i < N; ++i) {
            o.x[i] = double(px[k * N + i]);
            o.y[i] = double(py[k * N + i]);
            o.theta[i] = double(pt[k * N + i]);
        }
        o.collisions = coll[k];
        o.qp_infeasible = qpi[k];
        o.success = succ[k];
        o.scenario_metric = double(metric[k]);
        o.min_pairwise_distance = double(mind[k]);
        o.episode_return = double(ret[k]);
        auto TF = [&](int f) { return double(tf[static_cast<size_t>(f) * ctx->B + k]); };
        auto TI = [&](int w) { return ti[static_cast<size_t>(w) * ctx->B + k]; };
        auto TB = [&](int b) { return (TI(b >> 2) >> (8 * (b & 3))) & 0xff; };
        switch (c.task) {
            case MRSIM_TASK_NAVIGATION:
                for (int i = 0; i < N; ++i) { o.goals[i][0] = TF(2 * i); o.goals[i][1] = TF(2 * i + 1); }
                break;
            case MRSIM_TASK_PREDATOR_PREY:
                o.prey[0] = TF(0); o.prey[1] = TF(1); o.flash_timer = TI(0);
                break;
            case MRSIM_TASK_DISCOVERY:
                o.num_landmarks = y.discovery_num_landmarks;
                for (int q = 0; q < o.num_landmarks; ++q) {
                    o.landmarks[q][0] = TF(2 * q);
                    o.landmarks[q][1] = TF(2 * q + 1);
                    o.sensed[q] = (TI(0) >> q) & 1;
                    o.tagged[q] = (TI(1) >> q) & 1;
                }
                break;
            case MRSIM_TASK_RWARE: {
                const int S = y.rware_num_slots, R = mrsim_dev::rware_requests(y);
                o.num_slots = S;
                o.num_requests = R;
                for (int q = 0; q < S; ++q) o.slot_shelf[q] = TB(q);
                for (int i = 0; i < N; ++i) o.carried[i] = TB(S + i);
                for (int q = 0; q < R; ++q) o.requests[q] = TB(S + N + q);
                break;
            }
            case MRSIM_TASK_FORAGING:
                o.num_resources = y.foraging_num_resources;
                for (int q = 0; q < o.num_resources; ++q) {
                    o.resources[q][0] = TF(2 * q);
                    o.resources[q][1] = TF(2 * q + 1);
                    o.levels[q] = TI(1 + q);
                    o.foraged[q] = (TI(0) >> q) & 1;
                }
                break;
            case MRSIM_TASK_MATERIAL_TRANSPORT:
                o.circle_remaining = TF(0); o.rect_remaining = TF(1); o.delivered = TF(2); o.total_initial = TF(3);
                for (int i = 0; i < N; ++i) o.loads[i] = TF(4 + i);
                break;
            case MRSIM_TASK_ARCTIC_TRANSPORT:
                o.cols = y.arctic_grid_cols;
                o.rows = y.arctic_grid_rows;
                std::memcpy(o.goal_zone, y.arctic_goal_zone, sizeof o.goal_zone);
                for (int t = 0; t < o.cols * o.rows; ++t) o.tiles[t] = static_cast<int8_t>(TB(t));
                break;
            case MRSIM_TASK_WAREHOUSE:
                for (int i = 0; i < N; ++i) o.loaded[i] = (TI(0) >> i) & 1;
                break;
            case MRSIM_TASK_RANDOM_WAYPOINTS:
                for (int i = 0; i < N; ++i) {
                    o.targets[i][0] = TF(2 * i);
                    o.targets[i][1] = TF(2 * i + 1);
                    o.target_headings[i] = TF(2 * N + i);
                }
                break;
        }
    });
}

template <class Real>
void from_host_states(mrsim_ctx* ctx, const DevState<Real>& s, long long first, long long count,
                      const mrsim_env_state* in, cudaError_t* err) {
    const int N = ctx->N;
    const mrsim_cfg& c = ctx->cfg;
    const mrsim_layout& y = c.layout;
    DevState<Real> h;
    cudaError_t e = host_mirror<Real>(ctx, h);
    if (e != cudaSuccess) {
        *err = e;
        return;
    }
    Real *px = h.px + first * N, *py = h.py + first * N, *pt = h.pt + first * N;
    Real *metric = h.metric + first, *mind = h.min_dist + first, *ret = h.ep_return + first;
    int32_t *step = h.step_index + first, *coll = h.collisions + first, *qpi = h.qp_inf + first,
            *succ = h.success + first;
    uint64_t *key = h.key + first, *seed = h.seed + first, *pkey = h.pkey + first;
    int64_t* ep = h.episode + first;
    Real* tf = h.tf + first;
    int32_t* ti = h.ti + first;
    host_parallel_for(count, [&](long long k) {
        for (int f = 0; f < ctx->nf; ++f) tf[static_cast<size_t>(f) * ctx->B + k] = Real(0);
        for (int w = 0; w < ctx->ni; ++w) ti[static_cast<size_t>(w) * ctx->B + k] = 0;
        const mrsim_env_state& o = in[k];
        for (int i = 0; i < N; ++i) {
            px[k * N + i] = Real(o.x[i]);
            py[k * N + i] = Real(o.y[i]);
            pt[k * N + i] = Real(o.theta[i]);
        }
        step[k] = o.step_index;
        key[k] = o.rng_key;
        seed[k] = o.seed;
        pkey[k] = mrsim_dev::policy_key_of(o.seed);
        ep[k] = o.episode;
        coll[k] = static_cast<int32_t>(o.collisions);
        qpi[k] = static_cast<int32_t>(o.qp_infeasible);
        succ[k] = o.success;
        metric[k] = Real(o.scenario_metric);
        mind[k] = Real(o.min_pairwise_distance);
        ret[k] = Real(o.episode_return);
        auto TF = [&](int f, double v) { tf[static_cast<size_t>(f) * ctx->B + k] = Real(v); };
        auto TI = [&](int w, int v) { ti[static_cast<size_t>(w) * ctx->B + k] = v; };
        auto TB = [&](int b, int v) {
            int32_t& w = ti[static_cast<size_t>(b >> 2) * ctx->B + k];
            const int sh = 8 * (b & 3);
            w = (w & ~(0xff << sh)) | ((v & 0xff) << sh);
        };
        switch (c.task) {
            case MRSIM_TASK_NAVIGATION:
                for (int i = 0; i < N; ++i) { TF(2 * i, o.goals[i][0]); TF(2 * i + 1, o.goals[i][1]); }
                break;
            case MRSIM_TASK_PREDATOR_PREY:
                TF(0, o.prey[0]); TF(1, o.prey[1]); TI(0, o.flash_timer);
                break;
            case MRSIM_TASK_DISCOVERY: {
                int sm = 0, tg = 0;
                for (int q = 0; q < y.discovery_num_landmarks; ++q) {
                    TF(2 * q, o.landmarks[q][0]);
                    TF(2 * q + 1, o.landmarks[q][1]);
                    sm |= (o.sensed[q] ? 1 : 0) << q;
                    tg |= (o.tagged[q] ? 1 : 0) << q;
                }
                TI(0, sm);
                TI(1, tg);
                break;
            }
            case MRSIM_TASK_RWARE: {
                const int S = y.rware_num_slots, R = mrsim_dev::rware_requests(y);
                for (int q = 0; q < S; ++q) TB(q, o.slot_shelf[q]);
                for (int i = 0; i < N; ++i) TB(S + i, o.carried[i]);
                for (int q = 0; q < R; ++q) TB(S + N + q, o.requests[q]);
                break;
            }
            case MRSIM_TASK_FORAGING: {
                int fm = 0;
                for (int q = 0; q < y.foraging_num_resources; ++q) {
                    TF(2 * q, o.resources[q][0]);
                    TF(2 * q + 1, o.resources[q][1]);
                    TI(1 + q, o.levels[q]);
                    fm |= (o.foraged[q] ? 1 : 0) << q;
                }
                TI(0, fm);
                break;
            }
            case MRSIM_TASK_MATERIAL_TRANSPORT:
                TF(0, o.circle_remaining); TF(1, o.rect_remaining); TF(2, o.delivered); TF(3, o.total_initial);
                for (int i = 0; i < N; ++i) TF(4 + i, o.loads[i]);
                break;
            case MRSIM_TASK_ARCTIC_TRANSPORT:
                for (int t = 0; t < y.arctic_grid_cols * y.arctic_grid_rows; ++t) TB(t, o.tiles[t]);
                break;
            case MRSIM_TASK_WAREHOUSE: {
                int lm = 0;
                for (int i = 0; i < N; ++i) lm |= (o.loaded[i] ? 1 : 0) << i;
                TI(0, lm);
                break;
            }
            case MRSIM_TASK_RANDOM_WAYPOINTS:
                for (int i = 0; i < N; ++i) {
                    TF(2 * i, o.targets[i][0]);
                    TF(2 * i + 1, o.targets[i][1]);
                    TF(2 * N + i, o.target_headings[i]);
                }
                break;
        }
    });
    e = copy_state_slices<Real>(ctx, s, h, first, count, cudaMemcpyHostToDevice);
    *err = e;
}

// The feedforward policy's actions for the current state (ctx->ff set).
int run_policy(mrsim_ctx* ctx, int8_t* out, cudaStream_t s) {
    const cudaError_t e = ctx->fp64 ? policy_launch<double>(ctx, ctx->sd[ctx->cur], out, s)
                                    : policy_launch<float>(ctx, ctx->sf[ctx->cur], out, s);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "policy launch");
    return MRSIM_OK;
}


template <class Real>
cudaError_t capture_launch(mrsim_ctx* ctx, const DevState<Real>& st, const int8_t* actions, const uint8_t* done,
                           cudaStream_t s) {
    const long long total = ctx->B * ctx->N;
    const unsigned grid = static_cast<unsigned>((total + 255) / 256);
    mrsim_dev::capture_kernel<Real><<<grid, 256, 0, s>>>(st, actions, ctx->d_reward64, done, ctx->B, ctx->N,
                                                         ctx->d_cap + ctx->cap_steps * total);
    return cudaGetLastError();
}

// A step while capturing: materialise the policy's actions (when not given),
// step with a double team reward, then record (env, robot) rows of the new state.
int capture_step(mrsim_ctx* ctx, const int8_t* actions, float* obs, float* reward, uint8_t* done, float* next_obs,
                 cudaStream_t s) {
    if (ctx->cap_steps >= ctx->cap_max) return set_err(ctx, MRSIM_E_INVALID_ARGUMENT, "trajectory capture buffer full");
    CK(cudaSetDevice(ctx->device));
    const long long BN = ctx->B * ctx->N;
    if (!ctx->d_reward64) CK(ctx_malloc(ctx, &ctx->d_reward64, 8 * ctx->B));
    if (!ctx->d_done) CK(ctx_malloc(ctx, &ctx->d_done, ctx->B));
    if (!actions) {
        if (!ctx->d_pol_actions) CK(ctx_malloc(ctx, &ctx->d_pol_actions, BN));
        const bool dev_policy = ctx->ff || ctx->scripted;
        int rc = dev_policy ? run_policy(ctx, ctx->d_pol_actions, s) : MRSIM_OK;
        if (!dev_policy) {
            const unsigned grid = static_cast<unsigned>((BN + 255) / 256);
            if (ctx->fp64)
                mrsim_dev::random_actions_kernel<double><<<grid, 256, 0, s>>>(
                    ctx->sd[ctx->cur].step_index, ctx->sd[ctx->cur].pkey, ctx->N, ctx->B, ctx->d_pol_actions);
            else
                mrsim_dev::random_actions_kernel<float><<<grid, 256, 0, s>>>(
                    ctx->sf[ctx->cur].step_index, ctx->sf[ctx->cur].pkey, ctx->N, ctx->B, ctx->d_pol_actions);
            CK(cudaGetLastError());
        }
        if (rc != MRSIM_OK) return rc;
        actions = ctx->d_pol_actions;
    }
    uint8_t* dn = done ? done : ctx->d_done;
    int rc = ctx->fp64 ? do_step<double>(ctx, ctx->sd, actions, obs, reward, dn, next_obs, s, ctx->d_reward64)
                       : do_step<float>(ctx, ctx->sf, actions, obs, reward, dn, next_obs, s, ctx->d_reward64);
    if (rc != MRSIM_OK) return rc;
    const cudaError_t e = ctx->fp64 ? capture_launch<double>(ctx, ctx->sd[ctx->cur], actions, dn, s)
                                    : capture_launch<float>(ctx, ctx->sf[ctx->cur], actions, dn, s);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "capture launch");
    ctx->cap_steps += 1;
    return MRSIM_OK;
}
}  // namespace

extern "C" {

int mrsim_create(const mrsim_cfg* cfg, int device, int64_t num_envs, uint32_t flags, mrsim_ctx** out) {
    if (!cfg || !out || num_envs < 1) return MRSIM_E_INVALID_ARGUMENT;
    *out = nullptr;
    char msg[256] = {0};
    int rc = mrsim_config_validate(cfg, msg, sizeof msg);
    if (rc != MRSIM_OK) {
        std::fprintf(stderr, "mrsim_create: %s\n", msg);
        return rc;
    }
    mrsim_ctx* ctx = new mrsim_ctx;
    ctx->cfg = *cfg;
    ctx->device = device;
    ctx->B = num_envs;
    ctx->flags = flags;
    ctx->fp64 = (flags & MRSIM_FLAG_FP64) != 0;
    ctx->N = cfg->num_robots;
    ctx->n = 2 * ctx->N;
    ctx->P = ctx->N * (ctx->N - 1) / 2;
    ctx->D = mrsim_dev::obs_dim_of(*cfg);
    ctx->bdim = mrsim_dev::base_obs_dim(*cfg);
    mrsim_dev::task_fields(*cfg, &ctx->nf, &ctx->ni);
    ctx->var = mrsim_host::pick_variant(*cfg, flags);  // thread per env (N <= 4) or lane per robot
    ctx->L = ctx->var.L;
    cudaError_t e = cudaSetDevice(device);
    if (e != cudaSuccess) {
        rc = cuda_fail(ctx, e, "cudaSetDevice");
        std::fprintf(stderr, "mrsim_create: %s\n", ctx->last_error.c_str());
        delete ctx;
        return rc;
    }
    auto bail = [&](cudaError_t err, const char* where) {
        int code = cuda_fail(ctx, err, where);
        std::fprintf(stderr, "mrsim_create: %s\n", ctx->last_error.c_str());
        mrsim_destroy(ctx);
        return code;
    };
    cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, device);
    const size_t sb = ctx->fp64 ? state_bytes<double>(ctx->B, ctx->N, ctx->nf, ctx->ni)
                                : state_bytes<float>(ctx->B, ctx->N, ctx->nf, ctx->ni);
    for (int k = 0; k < 2; ++k) {
        if ((e = ctx_malloc(ctx, &ctx->mem[k], sb)) != cudaSuccess) return bail(e, "cudaMalloc state");
        cudaMemset(ctx->mem[k], 0, sb);
        if (kStateGuard) {
            std::vector<size_t> gaps;
            if (ctx->fp64) state_guards<double>(ctx->B, ctx->N, ctx->nf, ctx->ni, gaps);
            else state_guards<float>(ctx->B, ctx->N, ctx->nf, ctx->ni, gaps);
            for (size_t off : gaps) cudaMemset(static_cast<char*>(ctx->mem[k]) + off, 0xA5, kStateGuard);
        }
        if (ctx->fp64) carve_state(ctx->mem[k], ctx->B, ctx->N, ctx->nf, ctx->ni, ctx->sd[k]);
        else carve_state(ctx->mem[k], ctx->B, ctx->N, ctx->nf, ctx->ni, ctx->sf[k]);
    }
    // stats + undo log (values before the last update) + update serial; 256-byte aligned arrays
    const size_t stb = 2 * (static_cast<size_t>(ctx->B) * (4 + 8 * 5 + 8 * 2) + 8 * 256) +
                       static_cast<size_t>(ctx->B) * 8 + 256;
    if ((e = ctx_malloc(ctx, &ctx->stats_mem, stb)) != cudaSuccess) return bail(e, "cudaMalloc stats");
    {
        char* p = static_cast<char*>(ctx->stats_mem);
        auto take = [&](size_t bytes) {
            char* r = p;
            p += (bytes + 255) & ~size_t(255);
            return r;
        };
        mrsim_dev::EnvStats& st = ctx->st;
        st.episodes = reinterpret_cast<int32_t*>(take(4 * ctx->B));
        st.ret = reinterpret_cast<double*>(take(8 * ctx->B));
        st.ret_sq = reinterpret_cast<double*>(take(8 * ctx->B));
        st.metric = reinterpret_cast<double*>(take(8 * ctx->B));
        st.success = reinterpret_cast<double*>(take(8 * ctx->B));
        st.min_dist = reinterpret_cast<double*>(take(8 * ctx->B));
        st.collisions = reinterpret_cast<int64_t*>(take(8 * ctx->B));
        st.qp_inf = reinterpret_cast<int64_t*>(take(8 * ctx->B));
        st.u_episodes = reinterpret_cast<int32_t*>(take(4 * ctx->B));
        st.u_ret = reinterpret_cast<double*>(take(8 * ctx->B));
        st.u_ret_sq = reinterpret_cast<double*>(take(8 * ctx->B));
        st.u_metric = reinterpret_cast<double*>(take(8 * ctx->B));
        st.u_success = reinterpret_cast<double*>(take(8 * ctx->B));
        st.u_min_dist = reinterpret_cast<double*>(take(8 * ctx->B));
        st.u_collisions = reinterpret_cast<int64_t*>(take(8 * ctx->B));
        st.u_qp_inf = reinterpret_cast<int64_t*>(take(8 * ctx->B));
        st.upd_serial = reinterpret_cast<long long*>(take(8 * ctx->B));
        cudaMemset(ctx->stats_mem, 0, stb);
        cudaMemset(st.upd_serial, 0xff, 8 * ctx->B);  // -1: no update yet
        std::vector<double> inf(ctx->B, INFINITY);
        cudaMemcpy(st.min_dist, inf.data(), 8 * ctx->B, cudaMemcpyHostToDevice);
    }
    // error word, its step serial, then the step kernel's two warp-task counters
    if ((e = ctx_malloc(ctx, &ctx->d_err, 64)) != cudaSuccess) return bail(e, "cudaMalloc err");
    ctx->d_err_serial = reinterpret_cast<long long*>(ctx->d_err + 1);
    ctx->d_ticket = reinterpret_cast<unsigned*>(ctx->d_err + 2);  // step kernel [2], scripted kernel [2]
    cudaMemset(ctx->d_ticket, 0, 16);
    ctx->d_exit = reinterpret_cast<unsigned*>(ctx->d_err + 4);
    cudaMemset(ctx->d_exit, 0, 4);
    const unsigned long long none = ~0ull;
    cudaMemcpy(ctx->d_err, &none, sizeof none, cudaMemcpyHostToDevice);
    cudaMemset(ctx->d_err_serial, 0xff, 8);
    if (ctx->L == 1) {  // one thread per env: a plain grid of 64-env blocks, obs staged per warp
        ctx->block = mrsim_dev::kEnvBlock;
        const int stage = 32 * ctx->N * ctx->D;
        ctx->obs_stage = stage <= mrsim_dev::kEnvObsStageMax ? stage : 0;
        ctx->smem_group = 0;
        ctx->grid = static_cast<int>((ctx->B + ctx->block - 1) / ctx->block);
        ctx->grid_staged = ctx->grid;
        int bps = 0;
        const int smem = 4 * ctx->obs_stage * (ctx->block / 32);
        e = ctx->fp64 ? dispatch_occ<double>(cfg->task, ctx->var, ctx->block, smem, &bps)
                      : dispatch_occ<float>(cfg->task, ctx->var, ctx->block, smem, &bps);
        if (e != cudaSuccess) return bail(e, "occupancy query");
        if ((e = cudaDeviceSynchronize()) != cudaSuccess) return bail(e, "create sync");
        *out = ctx;
        return MRSIM_OK;
    }
    // launch geometry: persistent grid of (SMs x resident blocks)
    ctx->smem_group =
        ctx->fp64 ? mrsim_dev::GroupSmem<double>::bytes(ctx->N, ctx->nf, ctx->ni, ctx->var.L, ctx->var.MP, ctx->var.MO)
                  : mrsim_dev::GroupSmem<float>::bytes(ctx->N, ctx->nf, ctx->ni, ctx->var.L, ctx->var.MP, ctx->var.MO);
    const int smem = ctx->smem_group * (ctx->block / ctx->L);
    int bps = 0;
    e = ctx->fp64 ? dispatch_occ<double>(cfg->task, ctx->var, ctx->block, smem, &bps)
                  : dispatch_occ<float>(cfg->task, ctx->var, ctx->block, smem, &bps);
    if (e != cudaSuccess) return bail(e, "occupancy query");
    if (bps < 1) bps = 1;
    // Warp-staged observation stores (one contiguous block per warp, full-line writes; what makes
    // zero-copy obs to pinned host memory efficient), used by host-buffer steps only. On when it
    // costs no occupancy, and also when it costs one of 4 resident blocks: the host link is then the
    // bound (e2e over direct stores: discovery N=6 +75 %, MT N=10 +28 %, foraging N=6) — except for
    // arctic_transport, whose QP-heavy step loses more to the missing block (-14 %). Otherwise each
    // env's obs are staged in its group's dead QP matrix (no extra smem): arctic N=10 +22 %, and
    // rware N=6 (3 -> 2 blocks with the warp stage) +8 % over the warp stage
    // (profiles/r02/ab_host_stage.log).
    int bps_staged = bps;
    {
        const int stage = (((32 / ctx->L) * ctx->N * ctx->D + 3) / 4) * 4;  // floats per warp (16-B multiple)
        const int smem2 = smem + 4 * stage * (ctx->block / 32);
        int bps2 = 0;
        e = ctx->fp64 ? dispatch_occ<double>(cfg->task, ctx->var, ctx->block, smem2, &bps2)
                      : dispatch_occ<float>(cfg->task, ctx->var, ctx->block, smem2, &bps2);
        if (e != cudaSuccess) return bail(e, "occupancy query");
        const bool free = bps2 >= bps;
        const bool worth = bps2 >= 3 && bps2 + 1 >= bps && cfg->task != MRSIM_TASK_ARCTIC_TRANSPORT;
        ctx->obs_stage = (free || worth) ? stage : 0;
        if (!free && worth) bps_staged = bps2;
        // otherwise stage each env's obs in its group's dead QP inverse-Gram matrix (no extra smem)
        const long long nd = static_cast<long long>(ctx->N) * ctx->D;
        ctx->obs_ws_ok = mrsim_dev::obs_ws_stage_task(cfg->task) && (nd % 2) == 0 &&
                         nd * 4 <= 4ll * ctx->N * ctx->N * (ctx->fp64 ? 8 : 4);
    }
    const long long gpb = ctx->block / ctx->L;
    const long long need = (ctx->B + gpb - 1) / gpb;
    const long long full = static_cast<long long>(ctx->num_sms) * bps;
    const long long full_staged = static_cast<long long>(ctx->num_sms) * bps_staged;
    ctx->grid = static_cast<int>(need < full ? need : full);
    ctx->grid_staged = static_cast<int>(need < full_staged ? need : full_staged);
    if ((e = cudaDeviceSynchronize()) != cudaSuccess) return bail(e, "create sync");
    *out = ctx;
    return MRSIM_OK;
}

#ifdef MRSIM_DEVICE_CHECKS
int mrsim_debug_check_guards(mrsim_ctx* ctx);
#endif

void mrsim_destroy(mrsim_ctx* ctx) {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
#ifdef MRSIM_DEVICE_CHECKS
    if (mrsim_debug_check_guards(ctx) == MRSIM_E_RUNTIME) {  // a guard was overwritten: fail the whole run
        std::fprintf(stderr, "MRSIM_DEVICE_CHECKS: %s\n", ctx->last_error.c_str());
        std::abort();
    }
#endif
    for (int k = 0; k < 2; ++k) cudaFree(ctx->mem[k]);
    cudaFree(ctx->stats_mem);
    cudaFree(ctx->d_err);
    cudaFree(ctx->d_actions32);
    cudaFree(ctx->d_obs);
    cudaFree(ctx->d_reward64);
    cudaFree(ctx->d_done);
    if (ctx->h_err) cudaFreeHost(ctx->h_err);
    if (ctx->h_state) cudaFreeHost(ctx->h_state);
    ctx_free(ctx, ctx->d_wT);
    ctx_free(ctx, ctx->d_bias);
    cudaFree(ctx->d_pol_actions);
    ctx_free(ctx, ctx->d_cap);
    delete ctx;
}

const char* mrsim_last_error(const mrsim_ctx* ctx) { return ctx ? ctx->last_error.c_str() : "null context"; }
int64_t mrsim_num_envs(const mrsim_ctx* ctx) { return ctx ? ctx->B : 0; }

int mrsim_reset_seeds(mrsim_ctx* ctx, const uint64_t* seeds, float* obs_dev, void* stream) {
    if (!ctx || !seeds) return set_err(ctx, MRSIM_E_INVALID_ARGUMENT, "reset_batch: seed list is empty");
    CK(cudaSetDevice(ctx->device));
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    uint64_t* d_seeds = nullptr;
    CK(cudaMalloc(&d_seeds, 8 * ctx->B));
    CK(cudaMemcpyAsync(d_seeds, seeds, 8 * ctx->B, cudaMemcpyHostToDevice, s));
    int rc = ctx->fp64 ? do_reset<double>(ctx, ctx->sd, d_seeds, 0, 0, obs_dev, s)
                       : do_reset<float>(ctx, ctx->sf, d_seeds, 0, 0, obs_dev, s);
    CK(cudaStreamSynchronize(s));
    cudaFree(d_seeds);
    if (rc != MRSIM_OK) return rc;
    ctx->has_episodes = false;
    ctx->reset_done = true;
    return check_device_error(ctx, false);
}

int mrsim_reset_episodes(mrsim_ctx* ctx, uint64_t root_seed, int64_t first_episode, int64_t episode_stride,
                         float* obs_dev, void* stream) {
    if (!ctx || first_episode < 0) return set_err(ctx, MRSIM_E_INVALID_ARGUMENT, "reset: bad episode range");
    CK(cudaSetDevice(ctx->device));
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    ctx->root_seed = root_seed;
    ctx->episode_stride = episode_stride > 0 ? episode_stride : ctx->B;
    int rc = ctx->fp64 ? do_reset<double>(ctx, ctx->sd, nullptr, root_seed, first_episode, obs_dev, s)
                       : do_reset<float>(ctx, ctx->sf, nullptr, root_seed, first_episode, obs_dev, s);
    CK(cudaStreamSynchronize(s));
    if (rc != MRSIM_OK) return rc;
    ctx->has_episodes = true;
    ctx->reset_done = true;
    return check_device_error(ctx, false);
}

int mrsim_step(mrsim_ctx* ctx, const int8_t* actions_dev, float* obs_dev, float* reward_dev, uint8_t* done_dev,
               float* next_obs_dev, void* stream) {
    if (!ctx) return MRSIM_E_INVALID_ARGUMENT;
    if (!ctx->reset_done) return set_err(ctx, MRSIM_E_INVALID_ARGUMENT, "step before reset");
    if ((ctx->flags & MRSIM_FLAG_AUTO_RESET) && !ctx->has_episodes)
        return set_err(ctx, MRSIM_E_INVALID_ARGUMENT, "auto-reset needs mrsim_reset_episodes (episode seeds)");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (ctx->d_cap) return capture_step(ctx, actions_dev, obs_dev, reward_dev, done_dev, next_obs_dev, s);
    if (!actions_dev && (ctx->ff || ctx->scripted)) {  // the producer before the step: the policy on device
        CK(cudaSetDevice(ctx->device));
        const int rc = run_policy(ctx, ctx->d_pol_actions, s);
        if (rc != MRSIM_OK) return rc;
        actions_dev = ctx->d_pol_actions;
    }
    return ctx->fp64 ? do_step<double>(ctx, ctx->sd, actions_dev, obs_dev, reward_dev, done_dev, next_obs_dev, s)
                     : do_step<float>(ctx, ctx->sf, actions_dev, obs_dev, reward_dev, done_dev, next_obs_dev, s);
}

int mrsim_rollout(mrsim_ctx* ctx, int num_steps, float* obs_dev, float* reward_dev, uint8_t* done_dev,
                  void* stream) {
    if (!ctx || num_steps < 1) return set_err(ctx, MRSIM_E_INVALID_ARGUMENT, "rollout: num_steps must be >= 1");
    if (!ctx->reset_done) return set_err(ctx, MRSIM_E_INVALID_ARGUMENT, "step before reset");
    if ((ctx->flags & MRSIM_FLAG_AUTO_RESET) && !ctx->has_episodes)
        return set_err(ctx, MRSIM_E_INVALID_ARGUMENT, "auto-reset needs mrsim_reset_episodes (episode seeds)");
    if (ctx->ff || ctx->scripted || ctx->d_cap || ctx->L == 1 || !ctx->fp64)
        return set_err(ctx, MRSIM_E_UNSUPPORTED,
                       "rollout: fp64, the harness random policy on the lane-group kernel, without capture");
    CK(cudaSetDevice(ctx->device));
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    cudaError_t e;
    if (ctx->fp64) {
        StepParams<double> p = step_params<double>(ctx, ctx->sd, nullptr, obs_dev, reward_dev, done_dev, nullptr,
                                                   nullptr, nullptr);
        p.n_steps = num_steps;
        p.obs_stage = 0;  // device buffers: direct stores (the staged path's smem is not reserved here)
        e = dispatch_step<double>(ctx->cfg.task, p, ctx->var, ctx->grid, ctx->block,
                                  ctx->smem_group * (ctx->block / ctx->L), s);
    } else {
        StepParams<float> p = step_params<float>(ctx, ctx->sf, nullptr, obs_dev, reward_dev, done_dev, nullptr,
                                                 nullptr, nullptr);
        p.n_steps = num_steps;
        p.obs_stage = 0;
        e = dispatch_step<float>(ctx->cfg.task, p, ctx->var, ctx->grid, ctx->block,
                                 ctx->smem_group * (ctx->block / ctx->L), s);
    }
    if (e != cudaSuccess) return cuda_fail(ctx, e, "rollout kernel launch");
    step_done(ctx);
    ctx->env_steps += ctx->B * (num_steps - 1);
    return MRSIM_OK;
}

int mrsim_sync(mrsim_ctx* ctx, void* stream) {
    if (!ctx) return MRSIM_E_INVALID_ARGUMENT;
    CK(cudaSetDevice(ctx->device));
    CK(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)));
    return check_device_error(ctx, true);
}

int mrsim_step_host(mrsim_ctx* ctx, const int32_t* actions_host, float* obs_host, double* reward_host,
                    uint8_t* done_host, void* stream) {
    if (!ctx || !actions_host) return MRSIM_E_INVALID_ARGUMENT;
    if (!ctx->reset_done) return set_err(ctx, MRSIM_E_INVALID_ARGUMENT, "step before reset");
    CK(cudaSetDevice(ctx->device));
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const long long BN = ctx->B * ctx->N;
    const size_t obs_bytes = sizeof(float) * BN * ctx->D;
    // pinned caller buffers are used in place by the kernel (zero-copy); pageable ones are staged
    const int32_t* act = mapped_alias(actions_host);
    float* obs = mapped_alias(obs_host);
    double* rew = mapped_alias(reward_host);
    uint8_t* done = mapped_alias(done_host);
    if (!act) {
        if (!ctx->d_actions32) CK(ctx_malloc(ctx, &ctx->d_actions32, 4 * BN));
        CK(cudaMemcpyAsync(ctx->d_actions32, actions_host, 4 * BN, cudaMemcpyHostToDevice, s));
        act = ctx->d_actions32;
    }
    if (obs_host && !obs) {
        if (!ctx->d_obs) CK(ctx_malloc(ctx, &ctx->d_obs, obs_bytes));
        obs = ctx->d_obs;
    }
    if (reward_host && !rew) {
        if (!ctx->d_reward64) CK(ctx_malloc(ctx, &ctx->d_reward64, 8 * ctx->B));
        rew = ctx->d_reward64;
    }
    if (done_host && !done) {
        if (!ctx->d_done) CK(ctx_malloc(ctx, &ctx->d_done, ctx->B));
        done = ctx->d_done;
    }
    // The reference's std::vector<int> goes up as is; validate_actions (batch.hpp:226-237) runs in the
    // step kernel (first offender in (env, robot) order wins), and a failing step is rolled back below.
    const bool zero_copy_obs = obs && obs != ctx->d_obs;
    // error word + serial: written into pinned memory by the step kernel's last warp (no copy
    // after the kernel); a sentinel left in place means it was not (env kernel): copy it
    if (!ctx->h_err) CK(cudaMallocHost(&ctx->h_err, 16));
    constexpr unsigned long long kUnwritten = ~0ull - 1;
    volatile unsigned long long* herr = ctx->h_err;
    herr[0] = kUnwritten;
    unsigned long long* err_dev = mapped_alias(ctx->h_err);
    const int rc = ctx->fp64 ? do_step<double>(ctx, ctx->sd, nullptr, obs, nullptr, done, nullptr, s, rew, act,
                                               zero_copy_obs, err_dev)
                             : do_step<float>(ctx, ctx->sf, nullptr, obs, nullptr, done, nullptr, s, rew, act,
                                              zero_copy_obs, err_dev);
    if (rc != MRSIM_OK) return rc;
    if (obs_host && obs == ctx->d_obs) CK(cudaMemcpyAsync(obs_host, obs, obs_bytes, cudaMemcpyDeviceToHost, s));
    if (reward_host && rew == ctx->d_reward64)
        CK(cudaMemcpyAsync(reward_host, rew, 8 * ctx->B, cudaMemcpyDeviceToHost, s));
    if (done_host && done == ctx->d_done) CK(cudaMemcpyAsync(done_host, done, ctx->B, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (herr[0] == kUnwritten) {
        CK(cudaMemcpy(ctx->h_err, ctx->d_err, 16, cudaMemcpyDeviceToHost));
        CK(cudaMemset(ctx->d_exit, 0, 4));  // in case a launch ended without its epilogue
    }
    return check_device_error(ctx, true, actions_host, ctx->h_err);
}

int mrsim_observe(mrsim_ctx* ctx, float* obs_dev, void* stream) {
    if (!ctx || !obs_dev) return MRSIM_E_INVALID_ARGUMENT;
    CK(cudaSetDevice(ctx->device));
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    cudaError_t e = ctx->fp64 ? dispatch_observe<double>(ctx, ctx->sd[ctx->cur], obs_dev, s)
                              : dispatch_observe<float>(ctx, ctx->sf[ctx->cur], obs_dev, s);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "observe kernel launch");
    return MRSIM_OK;
}

int mrsim_observe_host(mrsim_ctx* ctx, float* obs_host) {
    if (!ctx || !obs_host) return MRSIM_E_INVALID_ARGUMENT;
    CK(cudaSetDevice(ctx->device));
    const size_t obs_bytes = sizeof(float) * ctx->B * ctx->N * ctx->D;
    if (!ctx->d_obs) CK(ctx_malloc(ctx, &ctx->d_obs, obs_bytes));
    int rc = mrsim_observe(ctx, ctx->d_obs, nullptr);
    if (rc != MRSIM_OK) return rc;
    CK(cudaMemcpy(obs_host, ctx->d_obs, obs_bytes, cudaMemcpyDeviceToHost));
    return MRSIM_OK;
}

int mrsim_set_policy_random(mrsim_ctx* ctx) {
    if (!ctx) return MRSIM_E_INVALID_ARGUMENT;
    ctx->ff = false;
    ctx->scripted = 0;
    return MRSIM_OK;
}

int mrsim_set_policy_scripted(mrsim_ctx* ctx, int kind) {
    if (!ctx) return MRSIM_E_INVALID_ARGUMENT;
    if (kind != MRSIM_POLICY_SCRIPTED_GOAL && kind != MRSIM_POLICY_PREY_CHASER)
        return set_err(ctx, MRSIM_E_INVALID_ARGUMENT, "unknown scripted policy");
    if (kind == MRSIM_POLICY_PREY_CHASER && ctx->cfg.task != MRSIM_TASK_PREDATOR_PREY)
        return set_err(ctx, MRSIM_E_INVALID_ARGUMENT, "prey_chaser policy only applies to predator_prey");
    const double cell = 0.05;  // policy.hpp:253-255
    const int cols = static_cast<int>((2.0 * ctx->cfg.arena_half_width) / cell);
    const int rows = static_cast<int>((2.0 * ctx->cfg.arena_half_height) / cell);
    if (cols * rows > mrsim_dev::kGridMaxCells)
        return set_err(ctx, MRSIM_E_UNSUPPORTED, "scripted planner grid exceeds the device capacity");
    CK(cudaSetDevice(ctx->device));
    if (!ctx->d_pol_actions) CK(ctx_malloc(ctx, &ctx->d_pol_actions, ctx->B * ctx->N));
    ctx->ff = false;
    ctx->scripted = kind;
    return MRSIM_OK;
}

int mrsim_set_policy_feedforward(mrsim_ctx* ctx, int num_layers, const int32_t* dims, const int32_t* activation,
                                 const double* weights, int greedy) {
    if (!ctx) return MRSIM_E_INVALID_ARGUMENT;
    const int IA = MRSIM_E_INVALID_ARGUMENT;
    // FeedforwardWeights::validate (policy.hpp:77-93)
    if (num_layers <= 0 || !dims || !activation || !weights) return set_err(ctx, IA, "weights: no layers");
    if (num_layers > MRSIM_POLICY_MAX_LAYERS)
        return set_err(ctx, MRSIM_E_UNSUPPORTED, "device policy supports <= 8 layers");
    mrsim_dev::PolicyNet net{};
    net.num_layers = num_layers;
    net.greedy = greedy ? 1 : 0;
    long long wsz = 0, bsz = 0;
    for (int l = 0; l < num_layers; ++l) {
        const int in = dims[2 * l], out = dims[2 * l + 1];
        if (in <= 0 || out <= 0) return set_err(ctx, IA, "weights: bad layer dimensions");
        if (l > 0 && dims[2 * l - 1] != in) return set_err(ctx, IA, "weights: layer dimensions do not chain");
        if (activation[l] < MRSIM_ACT_RELU || activation[l] > MRSIM_ACT_IDENTITY)
            return set_err(ctx, IA, "weights: unknown activation");
        if (in > MRSIM_POLICY_MAX_WIDTH || out > MRSIM_POLICY_MAX_WIDTH)
            return set_err(ctx, MRSIM_E_UNSUPPORTED, "device policy supports layer widths <= 256");
        net.in[l] = in;
        net.out[l] = out;
        net.act[l] = activation[l];
        net.w_off[l] = wsz;
        net.b_off[l] = bsz;
        wsz += static_cast<long long>(in) * out;
        bsz += out;
    }
    if (net.out[num_layers - 1] != 5) return set_err(ctx, IA, "weights: final layer must emit 5 logits");
    if (net.in[0] != ctx->D)  // FeedforwardWeights::forward size check (policy.hpp:96-99)
        return set_err(ctx, IA, "feedforward: observation size " + std::to_string(ctx->D) +
                                    " does not match expected " + std::to_string(net.in[0]));
    // transpose W (out x in) -> [in][out] per layer; split the biases out
    std::vector<double> wT(static_cast<size_t>(wsz)), bias(static_cast<size_t>(bsz));
    const double* src = weights;
    for (int l = 0; l < num_layers; ++l) {
        const int in = net.in[l], out = net.out[l];
        for (int o = 0; o < out; ++o)
            for (int i = 0; i < in; ++i) wT[net.w_off[l] + static_cast<long long>(i) * out + o] = src[o * in + i];
        src += static_cast<long long>(in) * out;
        for (int o = 0; o < out; ++o) bias[net.b_off[l] + o] = src[o];
        src += out;
    }
    CK(cudaSetDevice(ctx->device));
    CK(cudaDeviceSynchronize());
    ctx_free(ctx, ctx->d_wT);
    ctx_free(ctx, ctx->d_bias);
    ctx->d_wT = nullptr;
    ctx->d_bias = nullptr;
    ctx->ff = false;
    CK(ctx_malloc(ctx, &ctx->d_wT, sizeof(double) * wT.size()));
    CK(ctx_malloc(ctx, &ctx->d_bias, sizeof(double) * bias.size()));
    CK(cudaMemcpy(ctx->d_wT, wT.data(), sizeof(double) * wT.size(), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(ctx->d_bias, bias.data(), sizeof(double) * bias.size(), cudaMemcpyHostToDevice));
    if (!ctx->d_pol_actions) CK(ctx_malloc(ctx, &ctx->d_pol_actions, ctx->B * ctx->N));
    ctx->net = net;
    ctx->ff = true;
    ctx->scripted = 0;
    return MRSIM_OK;
}

int mrsim_policy_actions(mrsim_ctx* ctx, int8_t* actions_dev, void* stream) {
    if (!ctx || !actions_dev) return MRSIM_E_INVALID_ARGUMENT;
    if (!ctx->ff && !ctx->scripted) return mrsim_random_actions(ctx, actions_dev, stream);
    CK(cudaSetDevice(ctx->device));
    return run_policy(ctx, actions_dev, static_cast<cudaStream_t>(stream));
}

int mrsim_random_actions(mrsim_ctx* ctx, int8_t* actions_dev, void* stream) {
    if (!ctx || !actions_dev) return MRSIM_E_INVALID_ARGUMENT;
    CK(cudaSetDevice(ctx->device));
    const long long total = ctx->B * ctx->N;
    const int block = 256;
    const unsigned grid = static_cast<unsigned>((total + block - 1) / block);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (ctx->fp64)
        mrsim_dev::random_actions_kernel<double><<<grid, block, 0, s>>>(
            ctx->sd[ctx->cur].step_index, ctx->sd[ctx->cur].pkey, ctx->N, ctx->B, actions_dev);
    else
        mrsim_dev::random_actions_kernel<float><<<grid, block, 0, s>>>(
            ctx->sf[ctx->cur].step_index, ctx->sf[ctx->cur].pkey, ctx->N, ctx->B, actions_dev);
    CK(cudaGetLastError());
    return MRSIM_OK;
}

int mrsim_capture_begin(mrsim_ctx* ctx, int64_t max_steps) {
    if (!ctx || max_steps < 1) return MRSIM_E_INVALID_ARGUMENT;
    if (ctx->flags & MRSIM_FLAG_AUTO_RESET)
        return set_err(ctx, MRSIM_E_INVALID_ARGUMENT, "trajectory capture needs a context without auto-reset");
    CK(cudaSetDevice(ctx->device));
    CK(cudaDeviceSynchronize());
    ctx_free(ctx, ctx->d_cap);
    ctx->d_cap = nullptr;
    ctx->cap_max = ctx->cap_steps = 0;
    CK(ctx_malloc(ctx, &ctx->d_cap, sizeof(mrsim_traj_record) * max_steps * ctx->B * ctx->N));
    ctx->cap_max = max_steps;
    return MRSIM_OK;
}

int64_t mrsim_capture_steps(const mrsim_ctx* ctx) { return ctx ? ctx->cap_steps : 0; }

int mrsim_capture_read(mrsim_ctx* ctx, int64_t first_env, int64_t count, mrsim_traj_record* out) {
    if (!ctx || !out || !ctx->d_cap || first_env < 0 || count < 0 || first_env + count > ctx->B)
        return MRSIM_E_INVALID_ARGUMENT;
    CK(cudaSetDevice(ctx->device));
    CK(cudaDeviceSynchronize());
    const size_t rec = sizeof(mrsim_traj_record);
    const size_t width = rec * count * ctx->N, pitch = rec * ctx->B * ctx->N;
    CK(cudaMemcpy2D(out, width, ctx->d_cap + first_env * ctx->N, pitch, width, ctx->cap_steps,
                    cudaMemcpyDeviceToHost));
    return check_device_error(ctx, true);
}

int mrsim_capture_end(mrsim_ctx* ctx) {
    if (!ctx) return MRSIM_E_INVALID_ARGUMENT;
    CK(cudaSetDevice(ctx->device));
    CK(cudaDeviceSynchronize());
    ctx_free(ctx, ctx->d_cap);
    ctx->d_cap = nullptr;
    ctx->cap_max = ctx->cap_steps = 0;
    return MRSIM_OK;
}

int mrsim_get_env_states(mrsim_ctx* ctx, int64_t first, int64_t count, mrsim_env_state* out) {
    if (!ctx || !out || first < 0 || count < 0 || first + count > ctx->B) return MRSIM_E_INVALID_ARGUMENT;
    CK(cudaSetDevice(ctx->device));
    CK(cudaDeviceSynchronize());
    cudaError_t e = cudaSuccess;
    if (ctx->fp64) to_host_states<double>(ctx, ctx->sd[ctx->cur], first, count, out, &e);
    else to_host_states<float>(ctx, ctx->sf[ctx->cur], first, count, out, &e);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "download state");
    return MRSIM_OK;
}

int mrsim_set_env_states(mrsim_ctx* ctx, int64_t first, int64_t count, const mrsim_env_state* in) {
    if (!ctx || !in || first < 0 || count < 0 || first + count > ctx->B) return MRSIM_E_INVALID_ARGUMENT;
    for (int64_t k = 0; k < count; ++k)
        if (in[k].num_robots != ctx->N) return set_err(ctx, MRSIM_E_INVALID_ARGUMENT, "set_env_states: num_robots mismatch");
    CK(cudaSetDevice(ctx->device));
    CK(cudaDeviceSynchronize());
    cudaError_t e = cudaSuccess;
    if (ctx->fp64) from_host_states<double>(ctx, ctx->sd[ctx->cur], first, count, in, &e);
    else from_host_states<float>(ctx, ctx->sf[ctx->cur], first, count, in, &e);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "upload state");
    ctx->reset_done = true;
    return MRSIM_OK;
}

int mrsim_get_stats(mrsim_ctx* ctx, mrsim_stats* out) {
    if (!ctx || !out) return MRSIM_E_INVALID_ARGUMENT;
    CK(cudaSetDevice(ctx->device));
    CK(cudaDeviceSynchronize());
    const long long B = ctx->B;
    std::vector<int32_t> eps(B);
    std::vector<double> ret(B), ret2(B), met(B), suc(B), mind(B);
    std::vector<int64_t> col(B), qpi(B);
    CK(cudaMemcpy(eps.data(), ctx->st.episodes, 4 * B, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(ret.data(), ctx->st.ret, 8 * B, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(ret2.data(), ctx->st.ret_sq, 8 * B, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(met.data(), ctx->st.metric, 8 * B, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(suc.data(), ctx->st.success, 8 * B, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(mind.data(), ctx->st.min_dist, 8 * B, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(col.data(), ctx->st.collisions, 8 * B, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(qpi.data(), ctx->st.qp_inf, 8 * B, cudaMemcpyDeviceToHost));
    mrsim_stats s;
    std::memset(&s, 0, sizeof s);
    s.min_pairwise_distance = INFINITY;
    for (long long e = 0; e < B; ++e) {
        s.episodes += eps[e];
        s.sum_return += ret[e];
        s.sum_return_sq += ret2[e];
        s.sum_metric += met[e];
        s.sum_success += suc[e];
        s.sum_collisions += col[e];
        s.sum_qp_infeasible += qpi[e];
        s.min_pairwise_distance = std::fmin(s.min_pairwise_distance, mind[e]);
    }
    s.env_steps = ctx->env_steps;
    *out = s;
    return MRSIM_OK;
}

#ifdef MRSIM_DEVICE_CHECKS
// Checks builds only: verify every guard gap of both state copies and every allocation's guard
// tail still holds the fill pattern (an out-of-bounds device write lands in one of them).
int mrsim_debug_check_guards(mrsim_ctx* ctx) {
    if (!ctx) return MRSIM_E_INVALID_ARGUMENT;
    CK(cudaDeviceSynchronize());
    std::vector<unsigned char> buf(kStateGuard > kAllocGuard ? kStateGuard : kAllocGuard);
    auto bad = [&](size_t n) {
        for (size_t i = 0; i < n; ++i)
            if (buf[i] != 0xA5) return true;
        return false;
    };
    std::vector<size_t> gaps;
    if (ctx->fp64) state_guards<double>(ctx->B, ctx->N, ctx->nf, ctx->ni, gaps);
    else state_guards<float>(ctx->B, ctx->N, ctx->nf, ctx->ni, gaps);
    for (int k = 0; k < 2; ++k)
        for (size_t f = 0; f < gaps.size(); ++f) {
            CK(cudaMemcpy(buf.data(), static_cast<char*>(ctx->mem[k]) + gaps[f], kStateGuard, cudaMemcpyDeviceToHost));
            if (bad(kStateGuard))
                return set_err(ctx, MRSIM_E_RUNTIME, "guard overwritten: state copy " + std::to_string(k) +
                                                          " behind field " + std::to_string(f));
        }
    for (size_t t = 0; t < ctx->guard_tails.size(); ++t) {
        CK(cudaMemcpy(buf.data(), ctx->guard_tails[t].first, kAllocGuard, cudaMemcpyDeviceToHost));
        if (bad(kAllocGuard)) return set_err(ctx, MRSIM_E_RUNTIME, "guard overwritten: allocation tail " + std::to_string(t));
    }
    return MRSIM_OK;
}

// Checks builds only, negative control: overwrite the first byte of a guard (which = 0: the
// state guard behind field 0 of copy 0; 1: the first allocation tail) with `value` (0xA5 restores).
int mrsim_debug_poke_guard(mrsim_ctx* ctx, int which, int value) {
    if (!ctx || which < 0 || which > 1 || (which == 1 && ctx->guard_tails.empty())) return MRSIM_E_INVALID_ARGUMENT;
    std::vector<size_t> gaps;
    if (ctx->fp64) state_guards<double>(ctx->B, ctx->N, ctx->nf, ctx->ni, gaps);
    else state_guards<float>(ctx->B, ctx->N, ctx->nf, ctx->ni, gaps);
    char* at = which == 0 ? static_cast<char*>(ctx->mem[0]) + gaps[0] : ctx->guard_tails[0].first;
    CK(cudaMemset(at, value & 0xff, 1));
    CK(cudaDeviceSynchronize());
    return MRSIM_OK;
}
#endif

}  // extern "C"
