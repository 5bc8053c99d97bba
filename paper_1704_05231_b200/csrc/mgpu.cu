// Multi-GPU driver of the C ABI (SURVEY 8(b) fgb_mgpu_*, 8(e)): one process per
// GPU, the library owns an NCCL communicator.  The only collective is the one
// input broadcast from rank 0 (ncclBroadcast over NVLink / NVSwitch); every
// rank then computes its share into its own compact output -- no collective in
// the data path (the reference's only parallelism is the orientation thread
// pool, bank.py:77-87).
//
//   bank (config 5): the (frequency, direct k) units split into contiguous runs
//     per rank by an exact linear partition over a device-time model measured
//     on the B200, then a local-search refinement -- the same algorithm as
//     paper_1704_05231_b200/parallel.py:partition_units (a CPU test checks
//     both give identical partitions);
//   SDFT (config 4): conjugate u-pair heads {u, M-u} balanced by bin rows
//     (parallel.py:sdft_heads).
//
// NCCL is loaded with dlopen on first use (libnccl.so.2: torch's bundled copy
// when torch is loaded, else the system one), so the library itself has no
// link-time NCCL dependency.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "../../include/fgb200.h"

namespace {

// ---- device-time model, parallel.py:_FIT / run_cost (profiles/r02/unit_costs_c5.json) ----
// cost = A(h) + B1(h) single + B2(h) double (ms on an 8192^2 image), linear in h between the anchors
constexpr double kMpx = 67.108864;
constexpr double kFit[5][4] = {{6, 0.0553, 0.2141, 0.3204}, {12, 0.0329, 0.2401, 0.3043}, {24, 0.0701, 0.2338, 0.2985},
                                {48, 0.0638, 0.2936, 0.3483}, {96, 0.1561, 0.4585, 0.5044}};

double run_cost(double sigma, const std::vector<int>& ks, int n, double radius) {
    if (ks.empty()) return 0.0;
    const int h = std::max(1, (int)std::ceil(radius * sigma));
    double p[3] = {kFit[4][1], kFit[4][2], kFit[4][3]};
    if (h <= kFit[0][0]) {
        for (int j = 0; j < 3; ++j) p[j] = kFit[0][1 + j];
    } else {
        for (int i = 0; i < 4; ++i)
            if (h <= kFit[i + 1][0]) {
                const double w = (h - kFit[i][0]) / (kFit[i + 1][0] - kFit[i][0]);
                for (int j = 0; j < 3; ++j) p[j] = kFit[i][1 + j] + w * (kFit[i + 1][1 + j] - kFit[i][1 + j]);
                break;
            }
    }
    int single = 0;
    for (int k : ks) single += (k == 0 || 2 * k == n) ? 1 : 0;
    return (p[0] + p[1] * single + p[2] * ((int)ks.size() - single)) / kMpx;
}

// cost of one rank's unit list (units of one frequency share their row launches)
double part_cost(const std::vector<int>& p, const std::vector<double>& sigmas, int n, double radius) {
    const int nh = n / 2;
    std::map<int, std::vector<int>> runs;  // ordered by frequency; k sorted: parallel.py's summation order
    for (int u : p) runs[u / (nh + 1)].push_back(u % (nh + 1));
    double c = 0.0;
    for (auto& kv : runs) {
        std::sort(kv.second.begin(), kv.second.end());
        c += run_cost(sigmas[kv.first], kv.second, n, radius);
    }
    return c;
}

std::vector<std::vector<int>> partition_units(const std::vector<double>& sigmas, int n, int world, double radius) {
    const int nh = n / 2;
    std::vector<int> fo(sigmas.size());
    for (size_t i = 0; i < fo.size(); ++i) fo[i] = (int)i;
    std::stable_sort(fo.begin(), fo.end(), [&](int a, int b) { return sigmas[a] > sigmas[b] || (sigmas[a] == sigmas[b] && a < b); });
    std::vector<std::pair<int, int>> order;
    for (int i : fo)
        for (int k = 0; k <= nh; ++k) order.push_back({i, k});
    const int m = (int)order.size();
    world = std::max(1, std::min(world, m));
    auto seg_cost = [&](int a, int b) {
        std::vector<int> p;
        for (int j = a; j < b; ++j) p.push_back(order[j].first * (nh + 1) + order[j].second);
        return part_cost(p, sigmas, n, radius);
    };
    std::vector<std::vector<double>> cost(m + 1, std::vector<double>(m + 1, 0.0));
    for (int a = 0; a < m; ++a)
        for (int b = a + 1; b <= m; ++b) cost[a][b] = seg_cost(a, b);
    const double inf = HUGE_VAL;
    std::vector<std::vector<double>> best(world + 1, std::vector<double>(m + 1, inf));
    std::vector<std::vector<int>> cut(world + 1, std::vector<int>(m + 1, 0));
    best[0][0] = 0.0;
    for (int r = 1; r <= world; ++r)
        for (int b = 1; b <= m; ++b)
            for (int a = r - 1; a < b; ++a) {
                const double v = std::max(best[r - 1][a], cost[a][b]);
                if (v < best[r][b]) {
                    best[r][b] = v;
                    cut[r][b] = a;
                }
            }
    std::vector<std::pair<int, int>> bounds;
    for (int r = world, b = m; r > 0; --r) {
        const int a = cut[r][b];
        bounds.push_back({a, b});
        b = a;
    }
    std::reverse(bounds.begin(), bounds.end());
    std::vector<std::vector<int>> parts;
    for (auto& ab : bounds) {
        std::vector<int> p;
        for (int j = ab.first; j < ab.second; ++j) p.push_back(order[j].first * (nh + 1) + order[j].second);
        std::sort(p.begin(), p.end());
        parts.push_back(p);
    }
    // local search (parallel.py:_refine): move / swap units off the most loaded rank
    std::vector<double> pc;
    for (auto& p : parts) pc.push_back(part_cost(p, sigmas, n, radius));
    for (int round = 0; round < 200; ++round) {
        int r = 0;
        for (int j = 1; j < (int)parts.size(); ++j)
            if (pc[j] > pc[r]) r = j;
        const double top = pc[r];
        bool found = false;
        double bm = 0.0, ba = 0.0, bb = 0.0;
        int bq = -1;
        std::vector<int> bpa, bpb;
        for (int u : parts[r]) {
            std::vector<int> ru;
            for (int x : parts[r])
                if (x != u) ru.push_back(x);
            for (int q = 0; q < (int)parts.size(); ++q) {
                if (q == r) continue;
                std::vector<std::pair<std::vector<int>, std::vector<int>>> cand;
                std::vector<int> qu = parts[q];
                qu.push_back(u);
                cand.push_back({ru, qu});
                for (int v : parts[q]) {
                    std::vector<int> rv = ru, qv;
                    rv.push_back(v);
                    for (int x : parts[q])
                        if (x != v) qv.push_back(x);
                    qv.push_back(u);
                    cand.push_back({rv, qv});
                }
                for (auto& c : cand) {
                    const double a = part_cost(c.first, sigmas, n, radius), b = part_cost(c.second, sigmas, n, radius);
                    const double mx = std::max(a, b);
                    if (mx < top - 1e-12 && (!found || mx < bm - 1e-12)) {
                        found = true;
                        bm = mx;
                        bq = q;
                        ba = a;
                        bb = b;
                        bpa = c.first;
                        bpb = c.second;
                    }
                }
            }
        }
        if (!found) break;
        parts[r] = bpa;
        parts[bq] = bpb;
        pc[r] = ba;
        pc[bq] = bb;
    }
    for (auto& p : parts) std::sort(p.begin(), p.end());
    return parts;
}

std::vector<std::vector<int>> sdft_heads(int m, int world) {
    std::vector<int> heads;
    for (int u = 0; u <= m / 2; ++u) heads.push_back(u);
    auto w = [&](int u) { return (u == 0 || 2 * u == m) ? 1 : 2; };
    std::vector<int> order = heads;
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return w(a) > w(b) || (w(a) == w(b) && a < b); });
    std::vector<int> loads(world, 0);
    std::vector<std::vector<int>> parts(world);
    for (int u : order) {
        int r = 0;
        for (int j = 1; j < world; ++j)
            if (loads[j] < loads[r]) r = j;
        parts[r].push_back(u);
        loads[r] += w(u);
    }
    for (auto& p : parts) std::sort(p.begin(), p.end());
    return parts;
}

// ---- NCCL (dlopen) ----
struct Nccl {
    void* h = nullptr;
    ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
    const char* (*errorString)(ncclResult_t) = nullptr;
    bool load(std::string* err) {
        if (h) return true;
        for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
            h = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
            if (h) break;
        }
        if (!h) {
            *err = "libnccl.so.2 not found";
            return false;
        }
        getUniqueId = (decltype(getUniqueId))dlsym(h, "ncclGetUniqueId");
        commInitRank = (decltype(commInitRank))dlsym(h, "ncclCommInitRank");
        broadcast = (decltype(broadcast))dlsym(h, "ncclBroadcast");
        commDestroy = (decltype(commDestroy))dlsym(h, "ncclCommDestroy");
        errorString = (decltype(errorString))dlsym(h, "ncclGetErrorString");
        if (!getUniqueId || !commInitRank || !broadcast || !commDestroy || !errorString) {
            *err = "libnccl.so.2 lacks the expected symbols";
            h = nullptr;
            return false;
        }
        return true;
    }
};
Nccl g_nccl;
ncclComm_t g_comm = nullptr;
int g_world = 0, g_rank = -1, g_device = -1;
thread_local std::string g_merr;

int32_t merr(int32_t code, const std::string& m) {
    g_merr = m;
    return code;
}

}  // namespace

extern "C" {

const char* fgb_mgpu_last_error(void) { return g_merr.c_str(); }

int32_t fgb_mgpu_bank_units(const fgb_bank_desc* d, int32_t world, int32_t rank, int32_t* units, int32_t cap) {
    if (!d || !d->sigmas || d->n_freq < 1 || d->orientations < 1) return merr(FGB_EINVAL, "bad bank descriptor");
    if (world < 1 || rank < 0 || rank >= world) return merr(FGB_EINVAL, "rank must be in [0, world)");
    std::vector<double> sig(d->sigmas, d->sigmas + d->n_freq);
    const double radius = d->smoother.kind == FGB_SMOOTH_FIR ? d->smoother.radius : 3.0;
    const auto parts = partition_units(sig, d->orientations, world, radius);
    if (rank >= (int)parts.size()) return 0;  // more ranks than units: nothing for this one
    const auto& p = parts[rank];
    for (int i = 0; i < (int)p.size() && i < cap; ++i) units[i] = p[i];
    return (int32_t)p.size();
}

int32_t fgb_mgpu_sdft_heads(int32_t m, int32_t world, int32_t rank, int32_t* heads, int32_t cap) {
    if (m < 1 || world < 1 || rank < 0 || rank >= world) return merr(FGB_EINVAL, "bad SDFT shard arguments");
    const auto parts = sdft_heads(m, world);
    const auto& p = parts[rank];
    for (int i = 0; i < (int)p.size() && i < cap; ++i) heads[i] = p[i];
    return (int32_t)p.size();
}

int32_t fgb_mgpu_unique_id(unsigned char id[FGB_MGPU_ID_BYTES]) {
    std::string e;
    if (!g_nccl.load(&e)) return merr(FGB_EUNSUPPORTED, e);
    ncclUniqueId u;
    const ncclResult_t r = g_nccl.getUniqueId(&u);
    if (r != ncclSuccess) return merr(FGB_ENCCL, std::string("ncclGetUniqueId: ") + g_nccl.errorString(r));
    std::memcpy(id, u.internal, NCCL_UNIQUE_ID_BYTES);
    return FGB_OK;
}

int32_t fgb_mgpu_init(const unsigned char id[FGB_MGPU_ID_BYTES], int32_t world, int32_t rank, int32_t device) {
    if (world < 1 || rank < 0 || rank >= world) return merr(FGB_EINVAL, "rank must be in [0, world)");
    if (g_comm) return merr(FGB_EINVAL, "fgb_mgpu_init: already initialised (fgb_mgpu_finalize first)");
    std::string e;
    if (!g_nccl.load(&e)) return merr(FGB_EUNSUPPORTED, e);
    if (cudaSetDevice(device) != cudaSuccess) return merr(FGB_ECUDA, "cudaSetDevice failed");
    ncclUniqueId u;
    std::memcpy(u.internal, id, NCCL_UNIQUE_ID_BYTES);
    const ncclResult_t r = g_nccl.commInitRank(&g_comm, world, u, rank);
    if (r != ncclSuccess) {
        g_comm = nullptr;
        return merr(FGB_ENCCL, std::string("ncclCommInitRank: ") + g_nccl.errorString(r));
    }
    g_world = world;
    g_rank = rank;
    g_device = device;
    return FGB_OK;
}

int32_t fgb_mgpu_finalize(void) {
    if (g_comm) g_nccl.commDestroy(g_comm);
    g_comm = nullptr;
    g_world = 0;
    g_rank = -1;
    return FGB_OK;
}

static int32_t bcast_image(const fgb_image& im, void* img, cudaStream_t s) {
    const size_t es = im.dtype == FGB_F64 ? 8 : 4;
    const int64_t bs = im.batch > 1 ? im.batch_stride : (int64_t)im.height * im.pitch;
    const size_t n = (size_t)((int64_t)(im.batch - 1) * bs + (int64_t)(im.height - 1) * im.pitch + im.width);
    if (g_world == 1) return FGB_OK;
    const ncclResult_t r = g_nccl.broadcast(img, img, n * es, ncclUint8, 0, g_comm, s);
    if (r != ncclSuccess) return merr(FGB_ENCCL, std::string("ncclBroadcast: ") + g_nccl.errorString(r));
    return FGB_OK;
}

int32_t fgb_mgpu_bank(const fgb_bank_desc* d, void* img, void* out, void* stream) {
    if (!g_comm) return merr(FGB_EINVAL, "fgb_mgpu_bank: call fgb_mgpu_init first");
    if (!d || d->units) return merr(FGB_EINVAL, "fgb_mgpu_bank: descriptor must not carry a unit list");
    if (!d->reuse) return merr(FGB_EINVAL, "fgb_mgpu_bank: work units need reuse mode");
    cudaStream_t s = (cudaStream_t)stream;
    int32_t rc = bcast_image(d->img, img, s);
    if (rc != FGB_OK) return rc;
    std::vector<int32_t> units((size_t)d->n_freq * (d->orientations / 2 + 1));
    const int32_t nu = fgb_mgpu_bank_units(d, g_world, g_rank, units.data(), (int32_t)units.size());
    if (nu < 0) return nu;
    if (nu == 0) return FGB_OK;
    fgb_bank_desc dd = *d;
    dd.units = units.data();
    dd.n_units = nu;
    rc = fgb_bank(&dd, img, out, stream);
    if (rc != FGB_OK) return merr(rc, fgb_last_error());
    return FGB_OK;
}

int32_t fgb_mgpu_bank_entries(const fgb_bank_desc* d) {
    if (!g_comm) return merr(FGB_EINVAL, "fgb_mgpu_bank_entries: call fgb_mgpu_init first");
    std::vector<int32_t> units((size_t)d->n_freq * (d->orientations / 2 + 1));
    const int32_t nu = fgb_mgpu_bank_units(d, g_world, g_rank, units.data(), (int32_t)units.size());
    if (nu <= 0) return nu;
    fgb_bank_desc dd = *d;
    dd.units = units.data();
    dd.n_units = nu;
    return (int32_t)fgb_bank_entries(&dd);
}

int32_t fgb_mgpu_sdft(const fgb_sdft_desc* d, void* img, void* out, void* stream) {
    if (!g_comm) return merr(FGB_EINVAL, "fgb_mgpu_sdft: call fgb_mgpu_init first");
    if (!d || d->u_heads) return merr(FGB_EINVAL, "fgb_mgpu_sdft: descriptor must not carry a head list");
    cudaStream_t s = (cudaStream_t)stream;
    int32_t rc = bcast_image(d->img, img, s);
    if (rc != FGB_OK) return rc;
    std::vector<int32_t> heads(d->mx / 2 + 1);
    const int32_t nh = fgb_mgpu_sdft_heads(d->mx, g_world, g_rank, heads.data(), (int32_t)heads.size());
    if (nh < 0) return nh;
    if (nh == 0) return FGB_OK;
    fgb_sdft_desc dd = *d;
    dd.u_heads = heads.data();
    dd.n_heads = nh;
    rc = fgb_sdft(&dd, img, out, stream);
    if (rc != FGB_OK) return merr(rc, fgb_last_error());
    return FGB_OK;
}

}  // extern "C"
