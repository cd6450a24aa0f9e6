// Host side of the B200 Dykstra triangle sweep and the C ABI declared in
// include/metricproj_b200.h.
//
// One mp_handle = one solve session with device-resident state (the whole of
// PrimalState, DualStore and the instance; core.py:97-256).  A pass
// (run_pass, solver.py:166-210) is: snapshot -> one tile_round_kernel launch
// per round of the conflict-free schedule (the reference's barrier between
// rounds, solver.py:150-151, becomes the launch boundary) -> the fused pair
// phase + objective reductions -> a 1-CTA finalize -> ~64 bytes of stats to
// pinned host memory.  The sparse dual pools are double-buffered: pass k
// reads the pool pass k-1 wrote (SPEC.md "read pass k-1, write pass k").
#include <cuda.h>  // CUtensorMap (the encoder is resolved through the runtime)
#include <cuda_runtime.h>
#include <cub/device/device_radix_sort.cuh>
#include <dlfcn.h>
#include <nccl.h>  // types only: the functions are resolved at run time (nccl_api)

#include <algorithm>
#include <array>
#include <chrono>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <new>
#include <tuple>
#include <mutex>
#include <string>
#include <thread>
#include <atomic>
#include <vector>

#include "metricproj_b200.h"
#include "mp_aux.cuh"
#include "mp_device.cuh"
#include "mp_cube.cuh"
#include "mp_shard.cuh"

using namespace mp;


namespace {

thread_local std::string g_err;

// Experiment switches (launch-shape overrides such as MP_CLUSTER / MP_FORCE_C /
// MP_NO_TMA, the forced pool overflow MP_POOL_CAP0, timing toggles) exist only
// in -DMP_KNOBS builds: the `knobs` library variant that the shape-forcing
// tests and the tools/ A/B scripts load, and the diagnostic variants.  The
// product library reads two environment variables only: MP_NCCL_LIB (path of
// the NCCL library to dlopen) and MP_VERBOSE (planner log on stderr).
inline const char *knob(const char *name) {
#ifdef MP_KNOBS
    return getenv(name);
#else
    (void)name;
    return nullptr;
#endif
}

int fail(int code, const char *fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

// Device buffers of a finished session are kept for the next session of the
// same shape (repeated solve() calls: cudaMalloc/cudaFree of ~20 buffers cost
// milliseconds per session).  Only the handle destructor returns buffers,
// after synchronizing the session's stream; buffers are matched by exact size
// and device; at most 8 GiB are kept per process, and the cache is emptied
// and the allocation retried when cudaMalloc runs out of memory.
struct DevCache {
    std::mutex mu;
    std::multimap<std::pair<int, size_t>, void *> free_;
    std::map<void *, std::pair<int, size_t>> size_;
    size_t bytes = 0;
};
DevCache &dev_cache() {
    static DevCache *c = new DevCache();  // never destroyed: no frees after the driver unloads
    return *c;
}
cudaError_t dev_malloc(void **p, size_t sz) {
    int dev = 0;
    cudaGetDevice(&dev);
    DevCache &c = dev_cache();
    {
        std::lock_guard<std::mutex> lk(c.mu);
        auto it = c.free_.find({dev, sz});
        if (it != c.free_.end()) {
            *p = it->second;
            c.free_.erase(it);
            c.bytes -= sz;
            return cudaSuccess;
        }
    }
    cudaError_t e = cudaMalloc(p, sz);
    if (e == cudaErrorMemoryAllocation) {  // drop the cache and retry
        cudaGetLastError();
        std::lock_guard<std::mutex> lk(c.mu);
        for (auto &kv : c.free_) {
            c.size_.erase(kv.second);
            cudaFree(kv.second);
        }
        c.free_.clear();
        c.bytes = 0;
        e = cudaMalloc(p, sz);
    }
    if (e == cudaSuccess) {
        std::lock_guard<std::mutex> lk(c.mu);
        c.size_[*p] = {dev, sz};
    }
    return e;
}
// return a buffer to the cache (the caller has synchronized its users)
void dev_release(void *p) {
    if (!p) return;
    DevCache &c = dev_cache();
    std::lock_guard<std::mutex> lk(c.mu);
    auto it = c.size_.find(p);
    if (it == c.size_.end() || c.bytes + it->second.second > (size_t(8) << 30)) {
        if (it != c.size_.end()) c.size_.erase(it);
        cudaFree(p);
        return;
    }
    c.free_.insert({it->second, p});
    c.bytes += it->second.second;
}
// a buffer freed outside the destructor (pool growth) is really freed
cudaError_t dev_free(void *p) {
    if (!p) return cudaSuccess;
    DevCache &c = dev_cache();
    {
        std::lock_guard<std::mutex> lk(c.mu);
        c.size_.erase(p);
    }
    return cudaFree(p);
}
// Small pinned blocks (per-session stats) are recycled the same way.
std::mutex g_pin_mu;
std::vector<void *> g_pin_free;
constexpr size_t PIN_BLOCK = 256;
cudaError_t pin_malloc(void **p, size_t sz) {
    if (sz <= PIN_BLOCK) {
        std::lock_guard<std::mutex> lk(g_pin_mu);
        if (!g_pin_free.empty()) {
            *p = g_pin_free.back();
            g_pin_free.pop_back();
            return cudaSuccess;
        }
    }
    return cudaMallocHost(p, std::max(sz, PIN_BLOCK));
}
void pin_release(void *p) {
    if (!p) return;
    std::lock_guard<std::mutex> lk(g_pin_mu);
    if (g_pin_free.size() < 256) g_pin_free.push_back(p);
    else cudaFreeHost(p);
}
// First touch of a large output buffer on all host threads: a fresh numpy
// array costs ~28 ms of page faults per 64 MB when the driver's copy thread
// takes them one by one (measured on the GPU host); touching one byte per page
// from 16 threads beforehand takes a few ms.  The buffers are outputs, about to
// be overwritten.
void prefault_output(void *p, size_t bytes) {
    if (!p || bytes < (size_t(8) << 20)) return;
    const unsigned nthreads = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
    char *base = static_cast<char *>(p);
    std::vector<std::thread> pool;
    auto work = [&](unsigned q) {
        const size_t lo = bytes / nthreads * q, hi = q + 1 == nthreads ? bytes : bytes / nthreads * (q + 1);
        for (size_t o = lo; o < hi; o += 4096) base[o] = 0;
    };
    for (unsigned q = 1; q < nthreads; ++q) pool.emplace_back(work, q);
    work(0);
    for (auto &th : pool) th.join();
}

// Dual-pool capacity a previous session of the same shape grew to: the next
// one starts there (no re-allocation during its first passes, and its pool
// buffers come back from the cache).
std::mutex g_hint_mu;
std::map<std::tuple<int64_t, int, int, int64_t>, int32_t> g_pool_hint;
}  // namespace
#define cudaMalloc(p, sz) dev_malloc(reinterpret_cast<void **>(p), (sz))
#define cudaFree(p) dev_free(reinterpret_cast<void *>(p))
namespace {

#define NCK(call)                                                                     \
    do {                                                                              \
        ncclResult_t r_ = (call);                                                     \
        if (r_ != ncclSuccess)                                                        \
            return fail(MP_ERR_CUDA, "%s failed: %s", #call, nccl_api().errorString(r_)); \
    } while (0)

#define CK(call)                                                                        \
    do {                                                                                \
        cudaError_t e_ = (call);                                                        \
        if (e_ != cudaSuccess)                                                          \
            return fail(e_ == cudaErrorMemoryAllocation ? MP_ERR_OOM : MP_ERR_CUDA,     \
                        "%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_), __FILE__, \
                        __LINE__);                                                      \
    } while (0)

int64_t pair_count(int64_t n) { return n * (n - 1) / 2; }

int grid_for(int64_t work, int threads, int cap) {
    int64_t g = (work + threads - 1) / threads;
    if (g < 1) g = 1;
    if (g > cap) g = cap;
    return (int)g;
}

// Tile geometry (_kernels.py:74-86): rows [max(x,0), x+b-1], columns
// [max(z-b+1,0), z], middle [max(x+1,1), z-1]; level range of the tile.
TileDesc make_tile(int64_t x, int64_t z, int64_t b) {
    TileDesc t{};
    t.ilo = (int32_t)std::max<int64_t>(x, 0);
    t.ihi = (int32_t)(x + b - 1);
    t.klo = (int32_t)std::max<int64_t>(z - b + 1, 0);
    t.z = (int32_t)z;
    t.jlo = (int32_t)std::max<int64_t>(x + 1, 1);
    t.jhi = (int32_t)(z - 1);
    const int64_t j0 = std::max<int64_t>(t.jlo, t.ilo + 1);
    const int64_t k0 = std::max<int64_t>(t.klo, j0 + 1);
    t.Lbeg = (int32_t)(t.ilo + j0 + k0);
    t.Lend = (int32_t)(std::min<int64_t>(t.ihi, z - 2) + (z - 1) + z);
    return t;
}

// Tile bases of a pass in schedule order (schedule.tiled_rounds,
// schedule.py:117-153): per round the tiles (x + c*b, z - c*b).
void enumerate_tiles(int64_t n, int64_t b, std::vector<int64_t> &tx, std::vector<int64_t> &tz,
                     std::vector<int64_t> &round_cnt) {
    auto emit = [&](int64_t x, int64_t z) {
        int64_t cnt = 0;
        for (int64_t c = 0; std::max<int64_t>(x + c * b, 0) + 2 <= z - c * b; ++c) {
            tx.push_back(x + c * b);
            tz.push_back(z - c * b);
            ++cnt;
        }
        round_cnt.push_back(cnt);
    };
    for (int64_t z = n - 1; z >= 2; z -= b) emit(1 - b, z);
    for (int64_t x = 1; x + 2 <= n - 1; x += b) emit(x, n - 1);
}

// Triplets of tile (x, z) (Tile.size, schedule.py:36-67): sum over rows i and
// columns k >= i+2 of k-i-1.
int64_t tile_triplets(int64_t x, int64_t z, int64_t b) {
    const int64_t ilo = std::max<int64_t>(x, 0), ihi = x + b - 1, klo = std::max<int64_t>(z - b + 1, 0);
    int64_t s = 0;
    for (int64_t i = ilo; i <= ihi; ++i) {
        const int64_t a = std::max(klo, i + 2) - i - 1, c = z - i - 1;
        if (c >= a) s += (a + c) * (c - a + 1) / 2;
    }
    return s;
}

// Longest-processing-time assignment per round (distributed.shard_rounds):
// tiles by decreasing triplet count (ties: schedule position), each to the
// least-loaded rank (ties: lowest rank).
void lpt_owner(int64_t b, int world, const std::vector<int64_t> &tx, const std::vector<int64_t> &tz,
               const std::vector<int64_t> &round_cnt, std::vector<int32_t> &owner) {
    owner.assign(tx.size(), 0);
    int64_t off = 0;
    for (int64_t cnt : round_cnt) {
        std::vector<int64_t> idx((size_t)cnt), size((size_t)cnt);
        for (int64_t t = 0; t < cnt; ++t) {
            idx[(size_t)t] = t;
            size[(size_t)t] = tile_triplets(tx[(size_t)(off + t)], tz[(size_t)(off + t)], b);
        }
        std::stable_sort(idx.begin(), idx.end(),
                         [&](int64_t a, int64_t c) { return size[(size_t)a] > size[(size_t)c]; });
        std::vector<int64_t> load((size_t)world, 0);
        for (int64_t t : idx) {
            int g = 0;
            for (int r = 1; r < world; ++r)
                if (load[(size_t)r] < load[(size_t)g]) g = r;
            owner[(size_t)(off + t)] = g;
            load[(size_t)g] += size[(size_t)t];
        }
        off += cnt;
    }
}

// The tile that touches grid block (Ia, Kb) next after tile (I, K) in a pass
// (distributed.next_toucher; tests/test_distributed.py checks the closed form
// against the per-pair last toucher of the whole schedule).  Blocks and tiles
// share one grid: row block I = rows [1 + (I-1) b, I b] (0: row 0), column
// block K = columns [n - b - K b, n - 1 - K b].  The touchers of (Ia, Kb), in
// schedule order, are for Kb >= Ia the tiles (Ia, Ia..Kb), (Ia-1..0, Kb),
// (Ia, Ia-1..0), else (Kb..0, Kb), (Kb+1..Ia, Kb), (Ia, Kb-1..0); only the
// block's own tile (Ia, Kb) can be missing from the schedule.  Returns false
// when (I, K) is the block's last toucher of the pass.
template <class Exists>
bool next_toucher(int64_t Ia, int64_t Kb, int64_t I, int64_t K, Exists exists, int64_t &nI, int64_t &nK) {
    auto first = [&](int64_t i0, int64_t k0, bool have1, int64_t i1, int64_t k1) {
        if (exists(i0, k0)) {
            nI = i0, nK = k0;
            return true;
        }
        if (have1 && exists(i1, k1)) {
            nI = i1, nK = k1;
            return true;
        }
        return false;
    };
    const int64_t tail = Kb >= Ia ? Ia : Kb;  // the closing run (Ia, tail-1 .. 0) of the row
    if (I == Ia && K < tail) {
        if (K < 1) return false;
        nI = Ia, nK = K - 1;
        return true;
    }
    if (Kb >= Ia) {
        if (I == Ia) {  // opening run of the row, K in [Ia, Kb]
            if (K < Kb) return first(Ia, K + 1, Ia >= 1, Ia - 1, Kb);
            if (Ia < 1) return false;
            nI = Ia - 1, nK = Kb;
            return true;
        }
        if (I >= 1) {  // column run, I falling from Ia - 1 to 0
            nI = I - 1, nK = Kb;
            return true;
        }
        if (Ia < 1) return false;
        nI = Ia, nK = Ia - 1;
        return true;
    }
    if (I <= Kb && K == Kb) {  // column run of the first family, I falling
        if (I >= 1) {
            nI = I - 1, nK = Kb;
            return true;
        }
        return first(Kb + 1, Kb, Kb >= 1, Ia, Kb - 1);
    }
    if (K == Kb && I < Ia) return first(I + 1, Kb, Kb >= 1, Ia, Kb - 1);  // second family, I rising
    if (Kb < 1) return false;  // the block's own tile
    nI = Ia, nK = Kb - 1;
    return true;
}

// NCCL, resolved at run time so the library loads (and the CPU tests run)
// without it: prefer the copy already in the process (torch's), then
// $MP_NCCL_LIB, then the system libnccl.so.2.
struct NcclApi {
    ncclResult_t (*getUniqueId)(ncclUniqueId *) = nullptr;
    ncclResult_t (*commInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*send)(const void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*recv)(void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*allReduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t,
                              ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*groupStart)() = nullptr;
    ncclResult_t (*groupEnd)() = nullptr;
    const char *(*errorString)(ncclResult_t) = nullptr;
    std::string why;
};

const NcclApi &nccl_api() {
    static NcclApi api = [] {
        NcclApi a;
        void *lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (!lib && getenv("MP_NCCL_LIB")) lib = dlopen(getenv("MP_NCCL_LIB"), RTLD_NOW);
        if (!lib) lib = dlopen("libnccl.so.2", RTLD_NOW);
        if (!lib) {
            a.why = dlerror() ? dlerror() : "dlopen(libnccl.so.2) failed";
            return a;
        }
        a.getUniqueId = (decltype(a.getUniqueId))dlsym(lib, "ncclGetUniqueId");
        a.commInitRank = (decltype(a.commInitRank))dlsym(lib, "ncclCommInitRank");
        a.commDestroy = (decltype(a.commDestroy))dlsym(lib, "ncclCommDestroy");
        a.send = (decltype(a.send))dlsym(lib, "ncclSend");
        a.recv = (decltype(a.recv))dlsym(lib, "ncclRecv");
        a.allReduce = (decltype(a.allReduce))dlsym(lib, "ncclAllReduce");
        a.groupStart = (decltype(a.groupStart))dlsym(lib, "ncclGroupStart");
        a.groupEnd = (decltype(a.groupEnd))dlsym(lib, "ncclGroupEnd");
        a.errorString = (decltype(a.errorString))dlsym(lib, "ncclGetErrorString");
        if (!a.getUniqueId || !a.commInitRank || !a.commDestroy || !a.send || !a.recv || !a.allReduce ||
            !a.groupStart || !a.groupEnd || !a.errorString) {
            a.why = "libnccl.so.2 lacks a required symbol";
            a.getUniqueId = nullptr;
        }
        return a;
    }();
    return api;
}

}  // namespace

struct mp_handle {
    int dev = 0;
    cudaStream_t st = nullptr;
    int64_t n = 0, m = 0, ld = 0;
    int b = 0, kind = 0;
    uint32_t flags = 0;
    double eps = 0.0;
    bool unit_x = true, unit_f = true;
    StepConsts kc{};
    // max over rows of #{j : d_ij < 1/2} over its mean: hub rows (Chung-Lu
    // graphs) make the longest tiles of the small rounds exact-step bound
    double hub = 1.0;
    std::vector<int32_t> deg;  // #{j : d_ij < 1/2} per row (hub band split)

    // device state (x and winvx dense n x ld; the rest packed C(n,2))
    double *x = nullptr, *winvx = nullptr;
    double *f = nullptr, *d = nullptr, *w = nullptr, *regx = nullptr, *regf = nullptr,
           *winvf = nullptr, *pu = nullptr, *pl = nullptr, *tmp = nullptr;
    double *snap_x = nullptr, *snap_f = nullptr, *snap_pu = nullptr, *snap_pl = nullptr;

    // schedule; per round a launch shape: C CTAs (a thread-block cluster) per
    // tile, S slots per thread, NWC compute + NPW producer warps per CTA
    struct RoundCfg {
        int C = 1, S = 1, NWC = 1, NPW = 1, NT = 64, W = 128, RB = 1, LW = 32;
        int U = MP_BATCH;   // levels per batch (progress publish) of a compute warp
        int P = 1;          // WK row pitch in doubles (>= b: see round_shape)
        int PR = 128;       // WR row pitch in doubles (>= W)
        bool colm = false;  // column-major slots in each band
        size_t smem = 0;
        // row bands: band d owns tile rows [bst[d], bst[d+1]) with blw[d] lanes
        // per warp slot row (uniform RB-row bands unless a split is given)
        std::array<int, 17> bst{};
        std::array<int, 16> blw{};
    };
    std::vector<RoundCfg> rcfg;       // per round
    // Dataflow launch of the schedule's second family (mp_device.cuh, DF_*):
    // rounds [df_r0, end) run as one launch of df_cnt tiles with one shape
    // (rcfg of those rounds), each tile waiting on its two predecessors'
    // progress words instead of a launch boundary per round.
    bool df_allowed = true;           // off once sharded (per-round exchange)
    bool df_on = false;
    size_t df_r0 = 0;
    int64_t df_off = 0, df_cnt = 0;
    int4 *d_dep = nullptr;            // per dataflow tile: {row, column, diagonal} predecessor
    int32_t *d_prog = nullptr;        // per (dataflow tile, band) progress, then the claim counter
    int32_t tma_store = 1;            // box write-back of interior WK blocks (MP_NO_TMA_STORE: off)
    std::vector<int32_t> tile_round;  // round of each tile
    // schedule_kind "serial": the cube wavefront (mp_cube.cuh)
    std::vector<CubeDesc> cubes;          // all cubes, by cube level
    std::vector<int64_t> cube_off, cube_cnt;  // per cube level
    CubeDesc *d_cubes = nullptr;
    int64_t nb_cube = 0;                  // index blocks per axis
    std::vector<TileDesc> tiles;
    std::vector<int64_t> round_off, round_cnt;
    std::vector<int64_t> tile_x;      // tile base x per tile (for dual decode)
    std::vector<int32_t> tile_of_blk; // (iblock, kblock) -> tile index
    int64_t nib = 0, nkb = 0;
    TileDesc *d_tiles = nullptr;
    // 2-D TMA descriptors of x with box (b + 2t) x BLK, t = 0..7 (WK ring blocks
    // of row pitch b + 2t); null: element copies
    void *d_tmap[8] = {};
    int64_t nstreams = 0;

    // sparse duals: two pools, pool[rp] holds the previous pass's duals
    DualPool pool[2]{};
    int32_t pool_used[2] = {0, 0};
    int rp = 0;
    int64_t nnz = 0;

    // per-pass bookkeeping
    PassCounters *ctr = nullptr;
    double *partials = nullptr;
    int pair_grid = 1;
    DevStats *d_stats = nullptr, *h_stats = nullptr;
    cudaEvent_t ev[4]{};
    int64_t pass_index = 0;
    double metric_ms = 0.0, pair_ms = 0.0;
    int64_t launches = 0;
    unsigned long long *d_scan = nullptr;
    unsigned long long *trace = nullptr;  // mp_trace buffer (TR_NSLOTS counters)
    void *flush = nullptr;
    size_t flush_bytes = 0;

    // sharded execution (mp_shard; mp_shard.cuh)
    struct Shard {
        int world = 1, rank = 0;
        bool on = false, local = false;  // local: test transport (mp_group_run_passes)
        ncclComm_t comm = nullptr;
        std::vector<int32_t> owner;               // per tile
        std::vector<int64_t> my_off, my_cnt;      // per round, into d_my_tiles
        // next-toucher exchange (mp_shard.cuh): per round the pieces this rank
        // packs (grouped by destination) and unpacks (grouped by source), and
        // the values per peer segment of its send / receive buffer
        std::vector<int64_t> sp_off, sp_cnt, rp_off, rp_cnt;  // per round, into d_send_pc / d_recv_pc
        std::vector<int64_t> scnt, soff, rcnt, roff;          // per round x peer
        std::vector<char> round_any;                          // any rank sends anything after round r
        int64_t sent_per_pass = 0, recv_per_pass = 0;         // values (8 bytes each)
        TileDesc *d_my_tiles = nullptr;
        PieceDesc *d_send_pc = nullptr, *d_recv_pc = nullptr;
        double *sendbuf = nullptr, *recvbuf = nullptr;
        PassCounters *d_local = nullptr, *h_local = nullptr;  // this rank's counters
        int64_t local_nnz = 0;
    } sh;

    ~mp_handle() {
        if (dev >= 0) cudaSetDevice(dev);
        if (st) cudaStreamSynchronize(st);  // nothing in flight uses the buffers below
        double *bufs[] = {x, winvx, f, d, w, regx, regf, winvf, pu, pl, tmp,
                          snap_x, snap_f, snap_pu, snap_pl, partials};
        for (double *p : bufs) dev_release(p);
        for (auto &p : pool) {
            dev_release(p.rec);
            dev_release(p.head);
        }
        dev_release(d_tiles);
        dev_release(d_dep);
        dev_release(d_prog);
        for (void *t : d_tmap) dev_release(t);
        dev_release(d_cubes);
        dev_release(ctr);
        dev_release(d_stats);
        dev_release(d_scan);
        dev_release(trace);
        dev_release(flush);
        pin_release(h_stats);
        for (auto &e : ev)
            if (e) cudaEventDestroy(e);
        cudaFree(sh.d_my_tiles);
        cudaFree(sh.d_send_pc);
        cudaFree(sh.d_recv_pc);
        cudaFree(sh.sendbuf);
        cudaFree(sh.recvbuf);
        cudaFree(sh.d_local);
        if (sh.h_local) cudaFreeHost(sh.h_local);
        if (sh.comm) nccl_api().commDestroy(sh.comm);
        if (st) cudaStreamDestroy(st);
    }
};

namespace {

int alloc_pool(mp_handle *h, int which, int32_t cap) {
    {
        std::lock_guard<std::mutex> lk(g_hint_mu);
        int32_t &hint = g_pool_hint[{h->n, h->b, h->kind, h->nstreams}];
        hint = std::max(hint, cap);
    }
    DualPool &p = h->pool[which];
    cudaFree(p.rec);
    p.rec = nullptr;
    CK(cudaMalloc(&p.rec, (size_t)cap * sizeof(ChunkRec)));
    p.cap = cap;
    if (!p.head) {
        CK(cudaMalloc(&p.head, (size_t)std::max<int64_t>(h->nstreams, 1) * sizeof(int32_t)));
        CK(cudaMemsetAsync(p.head, 0xff, (size_t)std::max<int64_t>(h->nstreams, 1) * sizeof(int32_t),
                           h->st));
    }
    return MP_OK;
}

using TileKernel = void (*)(TileArgs);


template <int S>
TileKernel tile_kernel_s(int W, bool unit) {
    if (W == 256) return tile_round_kernel<S, 256, true>;  // W = 256 only for W = I
    return unit ? tile_round_kernel<S, 128, true> : tile_round_kernel<S, 128, false>;
}

// U: levels per batch (RoundCfg::U); short batches exist for the shape that
// needs them (2 slots per thread on the W = 256 ring, see round_shape)
TileKernel tile_kernel_for(int S, int W, bool unit, int U) {
    if (U == 4 && S == 2 && W == 256) return tile_round_kernel<2, 256, true, 4>;
    if (W == 512) return S == 1 ? tile_round_kernel<1, 512, true> : tile_round_kernel<2, 512, true>;
    switch (S) {
        case 1: return tile_kernel_s<1>(W, unit);
        case 2: return tile_kernel_s<2>(W, unit);
        case 3: return tile_kernel_s<3>(W, unit);
        case 4: return tile_kernel_s<4>(W, unit);
        default: return tile_kernel_s<5>(W, unit);
    }
}

cudaLaunchConfig_t tile_launch_config(const mp_handle::RoundCfg &c, int ntiles, cudaStream_t st,
                                      cudaLaunchAttribute *attr) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(ntiles * c.C), 1, 1);
    cfg.blockDim = dim3((unsigned)c.NT, 1, 1);
    cfg.dynamicSmemBytes = c.smem;
    cfg.stream = st;
    int na = 0;
    if (c.C > 1) {
        attr[na].id = cudaLaunchAttributeClusterDimension;
        attr[na].val.clusterDim.x = (unsigned)c.C;
        attr[na].val.clusterDim.y = 1;
        attr[na].val.clusterDim.z = 1;
        ++na;
    }
    if (!knob("MP_NO_PDL")) {  // programmatic dependent launch of consecutive rounds
        attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[na].val.programmaticStreamSerializationAllowed = 1;
        ++na;
    }
    cfg.attrs = attr;
    cfg.numAttrs = na;
    return cfg;
}

// Dynamic shared-memory opt-in of a kernel, set only when the size changes
// (a cudaFuncSetAttribute per round costs host time).  Setting the maximum
// once instead is much slower on the device (it changes the L1/shared split),
// so the exact size is kept.
int smem_optin(const void *k, size_t bytes) {
    static std::mutex mu;
    static std::vector<std::pair<std::pair<const void *, int>, size_t>> cur;
    std::lock_guard<std::mutex> lock(mu);
    int dev = 0;
    cudaGetDevice(&dev);
    for (auto &e : cur)
        if (e.first.first == k && e.first.second == dev) {
            if (e.second != bytes) {
                CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
                e.second = bytes;
            }
            return MP_OK;
        }
    CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
    // clusters of up to 16 CTAs (beyond the portable 8) in -DMP_CMAX=16 builds:
    // C = 10 / 14 bands were no faster than C = 8 at config 2
    if (MP_CMAX > 8) CK(cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    cur.push_back({{k, dev}, bytes});
    return MP_OK;
}

// One launch per round: ntiles tiles, C CTAs (one cluster) per tile.  The
// kernel's shared-memory opt-in is process-wide state: it is set and the
// launch issued under one lock, so sessions driven from several host threads
// (ctypes releases the GIL) cannot change it between the two.
std::mutex g_launch_mu;
int launch_tiles(mp_handle *h, const mp_handle::RoundCfg &c, const TileArgs &a, int ntiles) {
    TileKernel k = tile_kernel_for(c.S, c.W, h->unit_x, c.U);
    std::lock_guard<std::mutex> launch_lock(g_launch_mu);
    if (int rc = smem_optin((const void *)k, c.smem)) return rc;
    cudaLaunchAttribute attr[2];
    cudaLaunchConfig_t cfg = tile_launch_config(c, ntiles, h->st, attr);
    CK(cudaLaunchKernelEx(&cfg, k, a));
    return MP_OK;
}

// How many clusters of this shape the device can run at once (0 on error).
int max_active_clusters(const mp_handle *h, const mp_handle::RoundCfg &c) {
    TileKernel k = tile_kernel_for(c.S, c.W, h->unit_x, c.U);
    std::lock_guard<std::mutex> launch_lock(g_launch_mu);
    if (smem_optin((const void *)k, c.smem) != MP_OK) return 0;
    cudaLaunchAttribute attr[2];
    cudaLaunchConfig_t cfg = tile_launch_config(c, 1, h->st, attr);
    int n = 0;
    if (c.C == 1) {
        int per_sm = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, c.NT, c.smem) != cudaSuccess) return 0;
        int dev = 0, sms = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        return per_sm * sms;
    }
    if (cudaOccupancyMaxActiveClusters(&n, k, &cfg) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

// WK blocks can move as 2-D TMA boxes (tiled schedule, even b: box rows of
// b * 8 bytes, a multiple of 16)
bool tma_possible(const mp_handle *h) {
    return h->kind == 2 && !(h->b & 1) && h->b + 2 <= 256 && !knob("MP_NO_TMA");
}

// Shared-memory wavefronts per warp-wide 8-byte ring load (x_ij from WR
// with row pitch `pitch`, or x_jk from WK with row pitch `pitch`), averaged
// over the round's compute warps, slots and 16 consecutive levels: per
// half-warp, the most distinct addresses that share one of the 16 8-byte
// bank pairs.
double ring_waves(const mp_handle::RoundCfg &c, int b, int pitch, bool wk) {
    double tot = 0.0;
    int n = 0;
    for (int w = 0; w < std::min(c.NWC, 4); ++w)  // the lane map repeats with a shift
        for (int s = 0; s < c.S; ++s)
            for (int L = 0; L < 8; ++L) {
                for (int half = 0; half < 2; ++half) {
                    int64_t addr[16];
                    int na = 0;
                    for (int ln = 16 * half; ln < 16 * half + 16; ++ln) {
                        const int q = (w * c.S + s) * c.LW + ln;
                        if (ln >= c.LW || q >= c.RB * b) continue;
                        const int ii = c.colm ? q % c.RB : q / b, kk = c.colm ? q / c.RB : q % b;
                        const int jm = (4096 + L - ii - kk) & (c.W - 1);
                        const int64_t a = wk ? (int64_t)jm * pitch + kk : (int64_t)ii * pitch + jm;
                        bool dup = false;  // one address read by several lanes is a broadcast
                        for (int y = 0; y < na; ++y) dup |= addr[y] == a;
                        if (!dup) addr[na++] = a;
                    }
                    int cnt[16] = {}, worst = 0;
                    for (int x = 0; x < na; ++x) worst = std::max(worst, ++cnt[addr[x] & 15]);
                    tot += worst;
                }
                ++n;
            }
    return n ? tot / n : 0.0;
}

// Launch shape of a round with C CTAs per tile: the fewest slots per thread S
// with at most 15 compute warps (any S is correct: a warp waits until its
// predecessor finished the whole batch), up to 3 producer warps, W = 256
// ring when it fits.
mp_handle::RoundCfg round_shape(const mp_handle *h, int C, int lanes = -1,
                                const std::vector<int> *split = nullptr) {
    mp_handle::RoundCfg c;
    const int b = h->b;
    c.C = C;
    c.RB = (b + C - 1) / C;
    if (split) {  // non-uniform bands: the WR staging holds the largest band
        c.RB = 0;
        for (int d = 0; d < C; ++d) c.RB = std::max(c.RB, (*split)[(size_t)d + 1] - (*split)[(size_t)d]);
    }
    c.colm = C > 1;
    if (const char *e = knob("MP_COLMAJOR")) c.colm = atoi(e) != 0;
    const int slots = c.RB * b;
    int S = 1;
    if (const char *e = knob("MP_SLOTS")) S = std::max(S, atoi(e));
    // Column-major bands: a warp holds whole columns (LW a multiple of RB).  A
    // column split over two warps couples them through the in-column lattice
    // dependency and every exact step of the column stalls both (config 2, RB
    // = 5: LW = 30 is 8% faster than 32; 20 equals 30; 16 or 15 is slower).
    // Taken only when it needs no more slots per thread and leaves room for
    // three producer warps (else 32 lanes: config 3's C = 2 and C = 4 rounds).
    auto slots_per_thread = [&](int lw) {
        int s = S;
        while ((slots + lw * s - 1) / (lw * s) > MAX_CTA_THREADS / 32 - 1) ++s;
        return s;
    };
    c.LW = 32;
    if (c.colm && C > 1 && c.RB <= 32) {
        const int lw = c.RB * (32 / c.RB), s = slots_per_thread(lw);
        if (s <= slots_per_thread(32) && (slots + lw * s - 1) / (lw * s) <= MAX_CTA_THREADS / 32 - 3) c.LW = lw;
    }
    if (lanes < 0)
        if (const char *e = knob("MP_LANES")) lanes = atoi(e);
    if (lanes > 0 && C > 1) c.LW = std::max(1, std::min(32, lanes));  // cluster rounds only (one CTA needs them all)
    const int LW = c.LW;
    S = slots_per_thread(LW);
    c.S = S;
    c.NWC = (slots + LW * S - 1) / (LW * S);
    for (int d = 0; d <= 16; ++d) c.bst[(size_t)d] = std::min(d * c.RB, b);
    for (int d = 0; d < 16; ++d) c.blw[(size_t)d] = c.LW;
    if (split) {
        // every band's slots over the same warps, one slot per thread, its
        // columns spread evenly (band_lanes); a band too big for that is refused
        c.S = S = 1;
        c.NWC = MAX_CTA_THREADS / 32 - 2;
        if (const char *e = knob("MP_HUB_NWC")) c.NWC = std::max(1, std::min(MAX_CTA_THREADS / 32 - 1, atoi(e)));
        for (int d = 0; d <= C; ++d) c.bst[(size_t)d] = (*split)[(size_t)d];
        for (int d = C + 1; d <= 16; ++d) c.bst[(size_t)d] = b;
        for (int d = 0; d < C; ++d) {
            const int rows = c.bst[(size_t)d + 1] - c.bst[(size_t)d];
            c.blw[(size_t)d] = (rows * b + c.NWC - 1) / c.NWC;
            if (rows < 1 || c.blw[(size_t)d] > 32) c.S = MAX_SLOTS + 1;
        }
        if (c.S > MAX_SLOTS) return c;
    }
    c.NPW = std::min(3, MAX_CTA_THREADS / 32 - c.NWC);
    if (const char *e = knob("MP_PRODUCERS")) c.NPW = std::max(1, std::min(MAX_CTA_THREADS / 32 - c.NWC, atoi(e)));
    c.NT = 32 * (c.NWC + c.NPW);
    // ring width: as many j-slots as fit (a cluster's bands drift apart by up
    // to a few hundred levels; the ring bounds that drift)
    auto fits = [&](int W, int P, int PR) {
        return tile_smem_bytes(b, W, h->unit_x, c.NWC, c.RB, P, PR) <= 225 * 1024;
    };
    c.W = 128;
    if (h->unit_x && fits(256, b, 256)) c.W = 256;
    if (h->unit_x && C > 1 && S <= 2 && fits(512, b, 512)) c.W = 512;
    if (const char *e = knob("MP_RING_W")) c.W = std::min(c.W, std::max(128, atoi(e)));
    // Progress needs the ring to hold the slowest warp's whole j-window: the
    // producer frees blocks below slow - ihi - z and the warp reads up to
    // slow - ilo - klo, a span of 2b - 2, plus the block being loaded.  (b <=
    // 48 fits W = 128; larger tiles need W = 256, which only W = I has.)
    const int need_blocks = (2 * b - 2 + BLK) / BLK + 2;
    if (c.W / BLK < need_blocks) {  // no such shape: callers skip S > MAX_SLOTS
        c.S = MAX_SLOTS + 1;
        return c;
    }
    // Row pitches against bank conflicts: the lanes of a warp read x_ij at
    // WR[i][j % W] and x_jk at WK[j % W][k] with j = L - i - k, so with the
    // plain pitches (W, b) lanes with equal i + k (or equal i mod 2 when b =
    // 8 mod 16) share a bank.  Pick the pitches with the fewest shared-memory
    // wavefronts for this round's lane map (even pitches keep 16-byte pairs
    // aligned; a WK pitch > b is loaded as a wider TMA box and written back
    // element-wise).
    c.PR = c.W;
    if (!knob("MP_WR_PITCH_W")) {
        double best = 1e30;
        for (int pr = c.W; pr <= c.W + 14; pr += 2) {
            const double v = ring_waves(c, b, pr, false);
            if (v < best - 1e-9 && fits(c.W, b, pr)) best = v, c.PR = pr;
        }
    }
    c.P = b;
    if (!knob("MP_WK_PITCH_B")) {
        const int step = (b & 1) ? 1 : 2;
        const double plain = ring_waves(c, b, b, true);
        double best = 1e30;
        int bestp = b;
        for (int pk = b; pk <= b + 14 && pk <= 256; pk += step) {
            const double v = ring_waves(c, b, pk, true);
            if (v < best - 1e-9 && fits(c.W, pk, c.PR)) best = v, bestp = pk;
        }
        // a padded WK loses the box write-back of the last band: worth it only
        // when it at least halves the wavefronts (measured: RB = 5 at b = 40,
        // 5.6 -> 3.3 wavefronts, is a wash; RB >= 8, 8 -> 2, is not)
        if (best * 2.0 <= plain) c.P = bestp;
    }
    // Levels per batch: a warp trails its lattice predecessor by one batch, so a
    // tile's first warp runs (warps on the longest chain) x U levels ahead of
    // its last, and the ring must hold that plus a warp's own j-window (2b - 2),
    // the block in use and the blocks loaded ahead -- else the first warps stall
    // on slots the last ones still hold.  The 2-CTA shape on the W = 256 ring
    // (chain 2 + 13 warps, S = 2) does not fit with U = 8 (120 + 78 + 80 > 256;
    // timeline of a config-4 tile: every ~10th batch waits ~14,000 cycles for
    // the ring, 45% of the sweep) and runs U = 4 (config 4: 506 -> 474 ms/pass;
    // U = 6: 490; U = 2: 534; more slots per thread instead: 561 / 638).
    c.U = MP_BATCH;
    {
        const int chain = c.colm ? C + c.NWC : C * c.NWC;  // column-major bands: a 2-D grid of warps
        const int span = chain * MP_BATCH + 2 * b - 2 + BLK * (1 + MP_LOOKAHEAD);
        if (h->unit_x && c.S == 2 && c.W == 256 && span > c.W) c.U = 4;
    }
    if (const char *e = knob("MP_U")) {
        const int u = atoi(e);
        if (u == MP_BATCH || (u == 4 && h->unit_x && c.S == 2 && c.W == 256)) c.U = u;
    }
    c.smem = tile_smem_bytes(b, c.W, h->unit_x, c.NWC, c.RB, c.P, c.PR);
    return c;
}

// The shape every round can fall back to: one CTA per tile, or -- for tiles
// too big for one CTA (b > 48: more than MAX_SLOTS slots per thread) -- the
// smallest cluster that holds a tile (its rounds then run in waves).  C = 0:
// no shape fits.
mp_handle::RoundCfg fallback_shape(const mp_handle *h, int cmax) {
    const int b = h->b;
    for (int C = 1; C <= std::min(cmax, std::max(b, 1)); ++C) {
        if (C > 1 && (C - 1) * ((b + C - 1) / C) >= b) continue;
        const mp_handle::RoundCfg c = round_shape(h, C);
        if (c.S <= MAX_SLOTS && c.smem <= 227 * 1024) return c;
    }
    mp_handle::RoundCfg none;
    none.C = 0;
    return none;
}

// Row bands of balanced weight: the fewest-weight maximum over C bands of at
// most rmax rows each (binary search on the band weight, greedy bands), then
// the bands with the most rows split until there are C.  Returns the C + 1
// band starts, or an empty vector.
std::vector<int> balanced_split(const std::vector<double> &w, int C, int rmax) {
    const int b = (int)w.size();
    if (C < 1 || b < C || rmax < 1 || (int64_t)rmax * C < b) return {};
    auto greedy = [&](double T, std::vector<int> *out) {
        int bands = 0, r = 0;
        if (out) out->assign(1, 0);
        while (r < b) {
            double acc = 0.0;
            int rows = 0;
            while (r < b && rows < rmax && (rows == 0 || acc + w[(size_t)r] <= T)) acc += w[(size_t)r++], ++rows;
            ++bands;
            if (out) out->push_back(r);
        }
        return bands;
    };
    double lo = 0.0, hi = 0.0;
    for (double v : w) lo = std::max(lo, v), hi += v;
    for (int it = 0; it < 60; ++it) {
        const double mid = 0.5 * (lo + hi);
        if (greedy(mid, nullptr) <= C) hi = mid;
        else lo = mid;
    }
    std::vector<int> st;
    if (greedy(hi, &st) > C) return {};
    while ((int)st.size() - 1 < C) {
        int best = -1;
        for (int d = 0; d + 1 < (int)st.size(); ++d)
            if (st[(size_t)d + 1] - st[(size_t)d] >= 2 && (best < 0 || st[(size_t)d + 1] - st[(size_t)d] > st[(size_t)best + 1] - st[(size_t)best]))
                best = d;
        if (best < 0) return {};
        st.insert(st.begin() + best + 1, (st[(size_t)best] + st[(size_t)best + 1]) / 2);
    }
    return st;
}

// Launch shape per round: a round with few tiles spreads each tile over a
// cluster of C SMs (row bands, mp_device.cuh), as large as the device can
// co-schedule for all of the round's tiles at once (cnt[r] = tiles one
// device runs in round r: all of them, or one rank's share when sharded).
// Then one dual stream per (tile, band, compute warp), numbered in schedule
// order.
int plan_rounds(mp_handle *h, const std::vector<int64_t> &cnt_r) {
    const int b = h->b;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    int cmax = MP_CMAX;
    if (const char *e = knob("MP_CLUSTER")) cmax = std::max(1, std::min(MP_CMAX, atoi(e)));
    const mp_handle::RoundCfg one = fallback_shape(h, cmax);
    if (one.C == 0) return fail(MP_ERR_UNSUPPORTED, "tile size %d does not fit the device's launch shapes", b);
    int fb = 2;  // cluster size for rounds whose clusters do not all fit at once
    if (const char *e = knob("MP_WAVE_C")) fb = atoi(e);
    fb = std::min(fb, cmax);
    // Rounds of up to minc_cnt tiles get at least minc CTAs per tile, in waves
    // if need be: the longest tiles go first and their time is the round's
    // time.  Measured (pass 3): config 3 (Chung-Lu, hub rows in the longest
    // tiles) 167 -> 123 ms; config 4 (uniform) 586 -> 592 ms; config 5 -1%.
    // Larger rounds are throughput-bound and keep the largest fitting C.
    int minc = 6;
    if (const char *e = knob("MP_MIN_C")) minc = atoi(e);
    minc = std::min(minc, cmax);
    // Up to 3/8 of the SM count (55 on B200) for uniform instances (config 4:
    // 40-64 tiles equal, 72: +1%, 90: +4%); up to 2/3 (98) for hub instances,
    // whose longest tiles are exact-step bound and keep gaining from more CTAs
    // in larger rounds (config 5: 55 / 72 / 100 / 125 / 150 tiles 3.20 / 3.14 /
    // 3.06 / 3.06 / 3.13 s per pass; config 3's rounds hold at most 51).
    int64_t minc_cnt = h->hub >= 8.0 ? sms * 2 / 3 : sms * 3 / 8;
    if (const char *e = knob("MP_MIN_C_CNT")) minc_cnt = atoll(e);
    // Hub instances (h->hub >= 8): the small rounds' longest tiles hold the
    // hub rows and are exact-step bound; 8 bands of few-lane warps (the
    // fewest lanes, whole band columns, with <= 14 compute warps) spread a
    // row's exact steps over more warps.  Measured, config 3 (hub 83):
    // 105.7 -> 95.3 ms/pass (C = 8 with 30 / 20 / 15 lanes: 104.4 / 98.9 /
    // 95.3); config 2 (hub 1.6) would lose 2% with it, so it stays off there.
    bool hubby = h->hub >= 8.0 && !knob("MP_NO_HUB");
    mp_handle::RoundCfg hub_shape;
    if (hubby) {
        int C = std::min(8, std::min(cmax, b));
        if (const char *e = knob("MP_HUB_C")) C = std::max(2, std::min(std::min(cmax, b), atoi(e)));
        const int RB = (b + C - 1) / C;
        int lw = 32;
        for (int l = RB; l <= 32; l += RB)
            if ((RB * b + l - 1) / l <= MAX_CTA_THREADS / 32 - 2) {
                lw = l;
                break;
            }
        if (const char *e = knob("MP_HUB_LANES")) lw = std::max(1, std::min(32, atoi(e)));
        hub_shape = round_shape(h, C, lw);
        hubby = C > 1 && (C - 1) * RB < b && hub_shape.S <= MAX_SLOTS && hub_shape.smem <= 227 * 1024;
        // Bands of balanced exact-step weight instead of RB rows each: the
        // small rounds' critical tiles hold rows 1..b (row band 1), whose
        // stored duals per row follow close-degree^1.5 (config 3, rows 1-3:
        // 14.9 / 10.5 / 6.9 % measured, 14.4 / 10.2 / 6.8 % from degrees), so
        // the hub rows get bands of their own (every tile of the launch uses
        // the same relative split).
        // (at most 6 rows a band keeps the W = 512 ring; measured, config 3:
        // uniform 5-row bands 92.4 ms/pass; rmax 6 with 14 / 13 / 12 compute
        // warps 83.3 / 86.4 / 86.1; rmax 7 or 8 (W = 256 then) 97.9 / 97.6)
        int rmax = 6;
        if (const char *e = knob("MP_HUB_RMAX")) rmax = atoi(e);
        if (hubby && rmax > 0 && (int64_t)h->deg.size() > b && !knob("MP_NO_HUB_SPLIT")) {
            std::vector<double> w((size_t)b);
            for (int r = 0; r < b; ++r) w[(size_t)r] = std::pow((double)std::max(h->deg[(size_t)r + 1], 1), 1.5);
            const std::vector<int> split = balanced_split(w, C, rmax);
            if (!split.empty()) {
                const mp_handle::RoundCfg sc = round_shape(h, C, lw, &split);
                if (sc.S <= MAX_SLOTS && sc.smem <= 227 * 1024) hub_shape = sc;
            }
        }
        if (hubby && getenv("MP_VERBOSE")) {
            fprintf(stderr, "[mp] hub bands:");
            for (int d = 0; d < C; ++d) fprintf(stderr, " [%d,%d) lw %d", hub_shape.bst[(size_t)d], hub_shape.bst[(size_t)d + 1], hub_shape.blw[(size_t)d]);
            fprintf(stderr, " W=%d RB=%d smem=%zu\n", hub_shape.W, hub_shape.RB, hub_shape.smem);
        }
    }
    std::vector<int> cap(17, -1);  // co-resident clusters per C (queried once)
    std::vector<mp_handle::RoundCfg> shape(17);  // launch shape per C (computed once)
    std::vector<bool> have(17, false);
    // A shape taken regardless of the round's tile count (waves) must still be
    // placeable: at least one such cluster fits the device (a MIG slice, an
    // MPS SM limit or a smaller part may not hold 6 or 8 CTAs of one cluster).
    auto placeable = [&](int C) {
        if (!have[C]) shape[C] = round_shape(h, C), have[C] = true;
        if (shape[C].S > MAX_SLOTS || shape[C].smem > 227 * 1024) return false;
        if (cap[C] < 0) cap[C] = max_active_clusters(h, shape[C]);
        return cap[C] >= 1;
    };
    if (hubby && max_active_clusters(h, hub_shape) < 1) hubby = false;
    h->rcfg.clear();
    for (size_t r = 0; r < cnt_r.size(); ++r) {
        const int64_t cnt = cnt_r[r];
        mp_handle::RoundCfg best = one;
        bool found = false;
        if (const char *e = knob("MP_FORCE_C")) {  // experiment: one C for every round, in waves if need be
            const int C = std::max(1, std::min(MP_CMAX, atoi(e)));
            if (C > 1 && (C - 1) * ((b + C - 1) / C) < b && placeable(C)) best = shape[C];
            h->rcfg.push_back(best);
            continue;
        }
        for (int C = std::min(cmax, b); C >= 2 && cnt > 0; --C) {
            const int RB = (b + C - 1) / C;
            if ((C - 1) * RB >= b || cnt * C > sms) continue;
            if (!have[C]) shape[C] = round_shape(h, C), have[C] = true;
            const mp_handle::RoundCfg &c = shape[C];
            if (c.S > MAX_SLOTS || c.smem > 227 * 1024) continue;
            if (cap[C] < 0) cap[C] = max_active_clusters(h, c);
            if (cap[C] >= cnt) {
                best = c;
                found = true;
                break;
            }
        }
        // small rounds: at least minc CTAs per tile (see minc above)
        if (hubby && cnt > 0 && cnt <= minc_cnt) {
            best = hub_shape;
        } else if (best.C < minc && cnt > 0 && cnt <= minc_cnt && (minc - 1) * ((b + minc - 1) / minc) < b &&
                   placeable(minc)) {
            best = shape[minc];
        }
        // More tiles than the device co-schedules as clusters: clusters of
        // `fb` CTAs in waves beat one CTA per tile in a single wave (the
        // longest tiles go first and set the round's time; configs 4 / 5:
        // 0.68 -> 0.62 s and 4.8 -> 3.4 s per pass with C = 2 in waves).
        if (!found && best.C == 1 && cnt > 0 && fb >= 2 && (fb - 1) * ((b + fb - 1) / fb) < b && placeable(fb))
            best = shape[fb];
        h->rcfg.push_back(best);
    }
    // Second family (x >= 1) as one dataflow launch: tiles of one round wait
    // only on the two predecessor tiles of the previous round, ring block by
    // ring block, so the family's barrier depth (~n^2/(2b) levels) shrinks to
    // ~2n (dataflow depth half the barrier depth; all of it here).
    h->df_on = false;
    if (h->df_allowed && h->kind == MP_SCHEDULE_TILED && !knob("MP_NO_DF")) {
        size_t r0 = cnt_r.size();
        for (size_t r = 0; r < cnt_r.size(); ++r)
            if (h->round_cnt[r] && h->tile_x[(size_t)h->round_off[r]] >= 1) {
                r0 = r;
                break;
            }
        int64_t ndf = 0;
        for (size_t r = r0; r < cnt_r.size(); ++r) ndf += h->round_cnt[r];
        // Cluster size: the launch is either chain-bound (each round's tiles
        // trail their predecessors by ~3b + 2 ring blocks of levels, plus the
        // longest tile) or throughput-bound (all tiles' levels times C SMs
        // over the device).  A tile's time per level falls about as 1/C and
        // its SM-time stays put, so the largest C whose SM-levels per SM stay
        // within the chain's levels wins; else C = 2.  Measured (ms/pass):
        // config 2 (169 tiles) 5.40 / 4.62 / 4.38 / 4.27 at C = 2 / 4 / 6 / 8,
        // config 3 (2550 tiles) 105.8 / 116.2 / 112.8 / 115.4.
        int64_t lev = 0, lmax = 0, nr = 0;
        for (size_t r = r0; r < cnt_r.size(); ++r) {
            nr += h->round_cnt[r] > 0;
            for (int64_t t = h->round_off[r]; t < h->round_off[r] + h->round_cnt[r]; ++t) {
                const int64_t l = h->tiles[(size_t)t].Lend - h->tiles[(size_t)t].Lbeg + 1;
                lev += l;
                lmax = std::max(lmax, l);
            }
        }
        const int64_t chain = nr * (3 * (int64_t)b + 2 * BLK) + lmax;
        int C = 2;
        for (int c = 8; c > 2; --c)
            if (lev * c <= chain * sms) {
                C = c;
                break;
            }
        C = std::min(C, std::min(cmax, b));
        if (const char *e = knob("MP_DF_C")) C = std::max(1, std::min(std::min(cmax, b), atoi(e)));
        while (C > 1 && (C - 1) * ((b + C - 1) / C) >= b) --C;
        if (r0 < cnt_r.size() && ndf > 0) {
            int lanes = 0;
            if (const char *e = knob("MP_DF_LANES")) lanes = atoi(e);
            const mp_handle::RoundCfg c = round_shape(h, C, lanes);
            if (c.S <= MAX_SLOTS && c.smem <= 227 * 1024 && max_active_clusters(h, c) >= 1) {
                for (size_t r = r0; r < cnt_r.size(); ++r) h->rcfg[r] = c;
                h->df_on = true;
                h->df_r0 = r0;
                h->df_off = h->round_off[r0];
                h->df_cnt = ndf;
            }
        }
    }
    if (getenv("MP_VERBOSE")) {
        std::vector<int> hist(17, 0);
        for (const auto &c : h->rcfg) hist[(size_t)c.C]++;
        fprintf(stderr, "[mp] n=%lld b=%d rounds by cluster size:", (long long)h->n, b);
        for (int C = 1; C <= 16; ++C)
            if (hist[(size_t)C]) {
                const mp_handle::RoundCfg c = round_shape(h, C);
                fprintf(stderr, " C=%d:%d (S=%d NWC=%d NT=%d W=%d P=%d PR=%d smem=%zu cap=%d)", C, hist[(size_t)C],
                        c.S, c.NWC, c.NT, c.W, c.P, c.PR, c.smem, C > 1 ? cap[(size_t)C] : -1);
            }
        fprintf(stderr, "\n");
    }
    int64_t acc = 0;
    for (size_t t = 0; t < h->tiles.size(); ++t) {
        const mp_handle::RoundCfg &c = h->rcfg[(size_t)h->tile_round[t]];
        h->tiles[t].stream0 = acc;
        acc += (int64_t)c.C * c.NWC;
        const uint64_t keys = (uint64_t)(h->tiles[t].Lend - h->tiles[t].Lbeg + 1) * (uint64_t)c.S * 96ull;
        if (keys >= 0xFFFFFF00ull) return fail(MP_ERR_UNSUPPORTED, "tile too deep for 32-bit dual keys");
    }
    h->nstreams = acc;
    if (h->df_on) {  // predecessors of every dataflow tile (-1: first family / none)
        const int64_t nkb = h->nkb;
        auto find = [&](int64_t x, int64_t z) -> int {
            if (x < 1 || z < 2) return -1;
            const int64_t iblk = (x + b - 1) / b, kblk = (h->n - 1 - z) / b;
            if (iblk >= h->nib || kblk >= nkb) return -1;
            const int32_t t = h->tile_of_blk[(size_t)(iblk * nkb + kblk)];
            if (t < 0 || t < h->df_off || t >= h->df_off + h->df_cnt) return -1;
            if (h->tile_x[(size_t)t] != x || h->tiles[(size_t)t].z != z) return -1;
            return (int)(t - h->df_off);
        };
        std::vector<int4> dep((size_t)h->df_cnt);
        for (int64_t i = 0; i < h->df_cnt; ++i) {
            const size_t t = (size_t)(h->df_off + i);
            const int64_t x = h->tile_x[t], z = h->tiles[t].z;
            // diagonal predecessor only near the diagonal (tests/test_dataflow.py)
            dep[(size_t)i] = make_int4(find(x, z - b), find(x - b, z), z - x <= 2 * b ? find(x - b, z - b) : -1, 0);
        }
        const int C = h->rcfg[h->df_r0].C;
        dev_release(h->d_dep);
        dev_release(h->d_prog);
        h->d_dep = nullptr;
        h->d_prog = nullptr;
        CK(cudaMalloc(&h->d_dep, dep.size() * sizeof(int4)));
        CK(cudaMemcpy(h->d_dep, dep.data(), dep.size() * sizeof(int4), cudaMemcpyHostToDevice));
        CK(cudaMalloc(&h->d_prog, ((size_t)h->df_cnt * C + 1) * sizeof(int32_t)));
    }
    return MP_OK;
}


int launch_pairs(mp_handle *h, const PairArgs &a) {
    if (h->unit_x && h->unit_f)
        pair_phase_kernel<true, true><<<h->pair_grid, 256, 0, h->st>>>(a);
    else if (h->unit_x)
        pair_phase_kernel<true, false><<<h->pair_grid, 256, 0, h->st>>>(a);
    else if (h->unit_f)
        pair_phase_kernel<false, true><<<h->pair_grid, 256, 0, h->st>>>(a);
    else
        pair_phase_kernel<false, false><<<h->pair_grid, 256, 0, h->st>>>(a);
    CK(cudaGetLastError());
    return MP_OK;
}

// 2-D TMA descriptor of the dense x (dims n x n, row pitch ld): WK ring blocks
// (BLK rows j x b columns k) move as one box each.  Needs b * 8 bytes to be a
// multiple of 16 (even b); otherwise (or with MP_NO_TMA) the tile kernel
// copies WK element by element.  The encoder comes from the driver through
// cudaGetDriverEntryPoint (no link-time libcuda dependency).
typedef CUresult (*encode_tiled_fn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *,
                                    const cuuint64_t *, const cuuint64_t *, const cuuint32_t *,
                                    const cuuint32_t *, CUtensorMapInterleave, CUtensorMapSwizzle,
                                    CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
int make_x_tmap(mp_handle *h) {
    if (!tma_possible(h)) return MP_OK;
    // resolved once per process (the lookup costs tens of milliseconds)
    static void *fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            fn = nullptr;
        cudaGetLastError();
    });
    if (!fn) return MP_OK;  // no encoder: element copies
    for (int t = 0; t < 8 && h->b + 2 * t <= 256; ++t) {
        const int pad = 2 * t;
        CUtensorMap map;
        // inner extent ld (not n): with an odd n the box loads fault at the row end
        const cuuint64_t dims[2] = {(cuuint64_t)h->ld, (cuuint64_t)h->n};
        const cuuint64_t strides[1] = {(cuuint64_t)h->ld * sizeof(double)};
        const cuuint32_t box[2] = {(cuuint32_t)(h->b + pad), (cuuint32_t)BLK};
        const cuuint32_t estr[2] = {1, 1};
        const CUresult r = ((encode_tiled_fn)fn)(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, h->x, dims, strides,
                                                 box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                                 CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                                                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) return fail(MP_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
        void *&dst = h->d_tmap[t];
        CK(cudaMalloc(&dst, sizeof(CUtensorMap)));
        // pageable source: the call returns once `map` has been staged
        CK(cudaMemcpyAsync(dst, &map, sizeof(CUtensorMap), cudaMemcpyHostToDevice, h->st));
    }
    return MP_OK;
}

// descriptor for WK row pitch p (box p x BLK), or null
const void *x_tmap(const mp_handle *h, int p) {
    const int t = (p - h->b) / 2;
    return (p - h->b) % 2 == 0 && t >= 0 && t < 8 ? h->d_tmap[t] : nullptr;
}

// the launch's row bands (RoundCfg::bst / blw) into the kernel arguments
void set_bands(TileArgs &ta, const mp_handle::RoundCfg &c) {
    for (int d = 0; d <= 16; ++d) ta.bst[d] = (uint8_t)std::min(c.bst[(size_t)d], 255);
    for (int d = 0; d < 16; ++d) ta.blw[d] = (uint8_t)c.blw[(size_t)d];
    ta.rbmax = c.RB;
}

TileArgs tile_args(mp_handle *h) {
    TileArgs ta{};
    ta.x = h->x;
    ta.winvx = h->winvx;
    ta.ld = h->ld;
    ta.b = h->b;
    ta.kc = h->kc;
    ta.trace = h->trace;
    ta.tl_round = knob("MP_TL_ROUND") ? atoi(knob("MP_TL_ROUND")) : -1;
    ta.tl_tile = knob("MP_TL_TILE") ? atoi(knob("MP_TL_TILE")) : 0;
    ta.eps = h->eps;
    ta.rp = h->pool[h->rp];
    ta.wp = h->pool[h->rp ^ 1];
    ta.ctr = h->ctr;
    return ta;
}

// Pass = begin, [serial levels | rounds (+ exchange when sharded)],
// [counter all-reduce when sharded], end.  Nothing here syncs the host.
int pass_begin(mp_handle *h) {
    CK(cudaMemsetAsync(h->ctr, 0, sizeof(PassCounters), h->st));
    if (h->df_on)  // dataflow launch: progress words and the claim counter
        CK(cudaMemsetAsync(h->d_prog, 0, ((size_t)h->df_cnt * h->rcfg[h->df_r0].C + 1) * sizeof(int32_t),
                           h->st));
    // snapshot for an overflow retry of this pass
    CK(cudaMemcpyAsync(h->snap_x, h->x, (size_t)h->n * h->ld * sizeof(double),
                       cudaMemcpyDeviceToDevice, h->st));
    CK(cudaMemcpyAsync(h->snap_f, h->f, h->m * sizeof(double), cudaMemcpyDeviceToDevice, h->st));
    CK(cudaMemcpyAsync(h->snap_pu, h->pu, h->m * sizeof(double), cudaMemcpyDeviceToDevice, h->st));
    CK(cudaMemcpyAsync(h->snap_pl, h->pl, h->m * sizeof(double), cudaMemcpyDeviceToDevice, h->st));
    CK(cudaEventRecord(h->ev[1], h->st));
    return MP_OK;
}

int pass_serial(mp_handle *h) {
    CubeArgs ca{};
    ca.x = h->x;
    ca.winvx = h->winvx;
    ca.ld = h->ld;
    ca.n = (int32_t)h->n;
    ca.rp = h->pool[h->rp];
    ca.wp = h->pool[h->rp ^ 1];
    ca.ctr = h->ctr;
    ca.kc = h->kc;
    const size_t smem = cube_smem_bytes(h->unit_x);
    auto k = h->unit_x ? cube_level_kernel<true> : cube_level_kernel<false>;
    CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    for (size_t s = 0; s < h->cube_cnt.size(); ++s) {
        if (!h->cube_cnt[s]) continue;
        ca.cubes = h->d_cubes + h->cube_off[s];
        k<<<(unsigned)h->cube_cnt[s], CUBE_WARPS * 32, smem, h->st>>>(ca);
    }
    CK(cudaGetLastError());
    return MP_OK;
}

// This rank's tiles of round r: one CTA per tile.
int pass_round(mp_handle *h, size_t r, TileArgs &ta) {
    if (h->df_on && r >= h->df_r0) {  // the second family: one dataflow launch
        if (r != h->df_r0) return MP_OK;
        const mp_handle::RoundCfg &c = h->rcfg[r];
        ta.tiles = h->d_tiles + h->df_off;
        ta.round_id = (int32_t)r;
        ta.lw = c.LW;
        ta.colm = c.colm ? 1 : 0;
        ta.nt = c.NT;
        ta.nwc = c.NWC;
        ta.wkp = c.P;
        ta.wrp = c.PR;
        ta.tmap = x_tmap(h, c.P);
        ta.tma_store = h->tma_store;
        set_bands(ta, c);
        ta.df = 1;
        ta.dep = h->d_dep;
        ta.prog = h->d_prog;
        ta.qctr = h->d_prog + (size_t)h->df_cnt * c.C;
        const int rc = launch_tiles(h, c, ta, (int)h->df_cnt);
        ta.df = 0;
        return rc;
    }
    const int64_t cnt = h->sh.on ? h->sh.my_cnt[r] : h->round_cnt[r];
    if (!cnt) return MP_OK;
    ta.tiles = h->sh.on ? h->sh.d_my_tiles + h->sh.my_off[r] : h->d_tiles + h->round_off[r];
    const mp_handle::RoundCfg &c = h->rcfg[r];
    ta.round_id = (int32_t)r;
    ta.lw = c.LW;
    ta.colm = c.colm ? 1 : 0;
    ta.nt = c.NT;
    ta.nwc = c.NWC;
    ta.wkp = c.P;
    ta.wrp = c.PR;
    ta.tmap = x_tmap(h, c.P);
    ta.tma_store = h->tma_store;
    set_bands(ta, c);
    return launch_tiles(h, c, ta, (int)cnt);
}

bool round_exchanges(const mp_handle *h, size_t r) {
    return h->sh.on && h->sh.world > 1 && h->sh.round_any[r];
}

int pass_pack(mp_handle *h, size_t r) {
    if (!h->sh.sp_cnt[r]) return MP_OK;
    piece_copy_kernel<true><<<(unsigned)h->sh.sp_cnt[r], 256, 0, h->st>>>(
        h->sh.d_send_pc + h->sh.sp_off[r], h->x, h->ld, h->sh.sendbuf);
    CK(cudaGetLastError());
    return MP_OK;
}

int pass_unpack(mp_handle *h, size_t r) {
    if (!h->sh.rp_cnt[r]) return MP_OK;
    piece_copy_kernel<false><<<(unsigned)h->sh.rp_cnt[r], 256, 0, h->st>>>(
        h->sh.d_recv_pc + h->sh.rp_off[r], h->x, h->ld, h->sh.recvbuf);
    CK(cudaGetLastError());
    return MP_OK;
}

// After round r: every rank's packed segments to the ranks of the next
// touchers.  NCCL: one group of point-to-point sends and receives on the
// session stream; local transport (test harness): device copies.
int pass_exchange(std::vector<mp_handle *> &hs, size_t r) {
    mp_handle *h0 = hs[0];
    const int world = h0->sh.world;
    if (h0->sh.local) {
        for (mp_handle *dst : hs)
            for (mp_handle *src : hs) {
                const int64_t cnt = src->sh.scnt[r * world + dst->sh.rank];
                if (src == dst || !cnt) continue;
                CK(cudaMemcpyAsync(dst->sh.recvbuf + dst->sh.roff[r * world + src->sh.rank],
                                   src->sh.sendbuf + src->sh.soff[r * world + dst->sh.rank],
                                   (size_t)cnt * sizeof(double), cudaMemcpyDeviceToDevice, h0->st));
            }
        return MP_OK;
    }
    const NcclApi &N = nccl_api();
    const auto &S = h0->sh;
    NCK(N.groupStart());
    for (int g = 0; g < world; ++g) {
        if (g == S.rank) continue;
        if (S.scnt[r * world + g])
            NCK(N.send(S.sendbuf + S.soff[r * world + g], (size_t)S.scnt[r * world + g], ncclFloat64, g, S.comm,
                       h0->st));
        if (S.rcnt[r * world + g])
            NCK(N.recv(S.recvbuf + S.roff[r * world + g], (size_t)S.rcnt[r * world + g], ncclFloat64, g, S.comm,
                       h0->st));
    }
    NCK(N.groupEnd());
    return MP_OK;
}

// Keep this rank's own counters (its duals) before the all-reduce.
int pass_keep_local(mp_handle *h) {
    CK(cudaMemcpyAsync(h->sh.d_local, h->ctr, sizeof(PassCounters), cudaMemcpyDeviceToDevice, h->st));
    return MP_OK;
}

int pass_end(mp_handle *h) {
    CK(cudaEventRecord(h->ev[2], h->st));
    PairArgs pa{};
    pa.x = h->x;
    pa.ld = h->ld;
    pa.f = h->f;
    pa.d = h->d;
    pa.w = h->w;
    pa.winvx = h->winvx;
    pa.winvf = h->winvf;
    pa.regx = h->regx;
    pa.regf = h->regf;
    pa.pu = h->pu;
    pa.pl = h->pl;
    pa.n = h->n;
    pa.m = h->m;
    pa.eps = h->eps;
    pa.partials = h->partials;
    pa.ctr = h->ctr;
    int rc = launch_pairs(h, pa);
    if (rc) return rc;
    finalize_kernel<<<1, 1024, 0, h->st>>>(h->partials, h->pair_grid, h->eps, h->ctr, h->d_stats);
    CK(cudaGetLastError());
    CK(cudaEventRecord(h->ev[3], h->st));
    CK(cudaMemcpyAsync(h->h_stats, h->d_stats, sizeof(DevStats), cudaMemcpyDeviceToHost, h->st));
    if (h->sh.on)
        CK(cudaMemcpyAsync(h->sh.h_local, h->sh.d_local, sizeof(PassCounters), cudaMemcpyDeviceToHost,
                           h->st));
    return MP_OK;
}

// Enqueue one pass of a group of sessions that solve one instance together:
// a single unsharded session, one NCCL rank (hs = {this rank}), or all ranks
// of a local group sharing one stream (test transport).
int enqueue_group_pass(std::vector<mp_handle *> &hs, PassCounters **d_ctrs) {
    mp_handle *h0 = hs[0];
    for (mp_handle *h : hs) {
        CK(cudaEventRecord(h->ev[0], h->st));
        int rc = pass_begin(h);
        if (rc) return rc;
    }
    if (h0->kind == MP_SCHEDULE_SERIAL) {
        int rc = pass_serial(h0);
        if (rc) return rc;
    }
    std::vector<TileArgs> ta;
    for (mp_handle *h : hs) ta.push_back(tile_args(h));
    for (size_t r = 0; r < h0->round_cnt.size(); ++r) {
        for (size_t g = 0; g < hs.size(); ++g) {
            int rc = pass_round(hs[g], r, ta[g]);
            if (rc) return rc;
        }
        if (!round_exchanges(h0, r)) continue;
        for (mp_handle *h : hs) {
            int rc = pass_pack(h, r);
            if (rc) return rc;
        }
        if (int rc = pass_exchange(hs, r)) return rc;
        for (mp_handle *h : hs) {
            int rc = pass_unpack(h, r);
            if (rc) return rc;
        }
    }
    if (h0->sh.on) {
        for (mp_handle *h : hs) {
            int rc = pass_keep_local(h);
            if (rc) return rc;
        }
        if (h0->sh.world > 1) {
            if (h0->sh.local) {
                reduce_counters_kernel<<<1, 32, 0, h0->st>>>(d_ctrs, (int)hs.size());
                CK(cudaGetLastError());
            } else {
                const NcclApi &N = nccl_api();
                PassCounters *c = h0->ctr;
                NCK(N.groupStart());
                NCK(N.allReduce(&c->viol_bits, &c->viol_bits, 1, ncclUint64, ncclMax, h0->sh.comm, h0->st));
                NCK(N.allReduce(&c->nnz, &c->nnz, 1, ncclUint64, ncclSum, h0->sh.comm, h0->st));
                NCK(N.allReduce(&c->overflow, &c->overflow, 1, ncclInt32, ncclMax, h0->sh.comm, h0->st));
                NCK(N.groupEnd());
            }
        }
    }
    for (mp_handle *h : hs) {
        int rc = pass_end(h);
        if (rc) return rc;
    }
    return MP_OK;
}

int restore_snapshot(mp_handle *h) {
    CK(cudaMemcpyAsync(h->x, h->snap_x, (size_t)h->n * h->ld * sizeof(double),
                       cudaMemcpyDeviceToDevice, h->st));
    CK(cudaMemcpyAsync(h->f, h->snap_f, h->m * sizeof(double), cudaMemcpyDeviceToDevice, h->st));
    CK(cudaMemcpyAsync(h->pu, h->snap_pu, h->m * sizeof(double), cudaMemcpyDeviceToDevice, h->st));
    CK(cudaMemcpyAsync(h->pl, h->snap_pl, h->m * sizeof(double), cudaMemcpyDeviceToDevice, h->st));
    return MP_OK;
}

int upload_packed(mp_handle *h, double **dst, const double *src) {
    CK(cudaMalloc(dst, h->m * sizeof(double)));
    CK(cudaMemcpyAsync(*dst, src, h->m * sizeof(double), cudaMemcpyHostToDevice, h->st));
    return MP_OK;
}

// decode one stored entry of tile t / warp w into the reference key
struct Decoded {
    int64_t i, j, k, kind;
};

// Index of cube (I, J, K), I <= J <= K, in h->cubes (cube levels in order,
// inside a level I then J ascending).
int64_t cube_index(const mp_handle *h, int64_t I, int64_t J, int64_t K) {
    const int64_t sl = I + J + K, nb = h->nb_cube;
    auto jlo = [&](int64_t i) { return std::max(i, sl - i - nb + 1); };  // J range of first index i
    auto jhi = [&](int64_t i) { return (sl - i) / 2; };
    int64_t t = h->cube_off[(size_t)sl];
    for (int64_t i = 0; i < I; ++i) t += std::max<int64_t>(0, jhi(i) - jlo(i) + 1);
    return t + (J - jlo(I));
}

// w = the stream's index within its tile: band * NWC + warp
Decoded decode_entry(const mp_handle *h, int64_t t, int w, uint32_t key) {
    const TileDesc &T = h->tiles[t];
    const mp_handle::RoundCfg &c = h->rcfg[(size_t)h->tile_round[(size_t)t]];
    const int band = w / c.NWC, wb = w % c.NWC;
    const uint32_t per_level = (uint32_t)c.S * 96u;
    const uint32_t lvl = key / per_level, rem = key % per_level;
    const int s = (int)(rem / 96u), r2 = (int)(rem % 96u);
    const int lane = r2 / 3, kind = r2 % 3;
    // a band's slot map covers its real rows (single-row tiles: band 0, 1 row)
    const int64_t nrows = (int64_t)T.ihi - T.ilo + 1;
    const int64_t r0 = c.bst[(size_t)band], r1 = std::min<int64_t>(h->b, c.bst[(size_t)band + 1]),
                  rbc = std::max<int64_t>(1, std::min<int64_t>(r1, nrows) - r0);
    const int64_t LW = band_lanes(c.blw[(size_t)band], c.NWC, c.S, (int)rbc, (int)(r1 - r0), h->b, c.colm);
    const int64_t q = ((int64_t)wb * c.S + s) * LW + lane;
    const int64_t ii = c.colm ? r0 + q % rbc : r0 + q / h->b;
    const int64_t kk = c.colm ? q / rbc : q % h->b;
    Decoded d;
    d.i = T.ilo + ii;
    d.k = T.klo + kk;
    d.j = (int64_t)T.Lbeg + lvl - d.i - d.k;
    d.kind = kind;
    return d;
}

}  // namespace

// ---------------------------------------------------------------------------
// C ABI
// ---------------------------------------------------------------------------
extern "C" {

const char *mp_last_error(void) { return g_err.c_str(); }

const char *mp_version(void) {
#ifdef MP_KNOBS
    return "metricproj_b200 0.2.0 (sm_100a, +knobs)";
#else
    return "metricproj_b200 0.2.0 (sm_100a)";
#endif
}

int mp_create(const mp_instance *inst, const mp_config *cfg, mp_handle **out) {
    g_err.clear();
    // MP_TIME_CREATE: wall time of the creation phases on stderr
    const bool tcr = knob("MP_TIME_CREATE") != nullptr;
    cudaStream_t tst = nullptr;
    auto tnow = [] {
        return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
    };
    double tc0 = tcr ? tnow() : 0.0;
    auto tmark = [&](const char *what) {
        if (!tcr) return;
        if (tst) cudaStreamSynchronize(tst);
        const double t = tnow();
        fprintf(stderr, "[mp] create %-14s %7.3f ms\n", what, t - tc0);
        tc0 = t;
    };
    if (!inst || !cfg || !out) return fail(MP_ERR_ARG, "null argument");
    *out = nullptr;
    const int64_t n = inst->n;
    if (n < 3) return fail(MP_ERR_ARG, "need n >= 3, got %lld", (long long)n);
    if (n > 2000000) return fail(MP_ERR_ARG, "n too large: %lld", (long long)n);
    if (!(inst->epsilon > 0.0) || !std::isfinite(inst->epsilon))
        return fail(MP_ERR_ARG, "epsilon must be positive, got %g", inst->epsilon);
    if (!inst->d_flat || !inst->w_flat) return fail(MP_ERR_ARG, "d_flat / w_flat are required");
    if (cfg->schedule_kind < 0 || cfg->schedule_kind > 2)
        return fail(MP_ERR_ARG, "unknown schedule_kind %d", cfg->schedule_kind);
    if (cfg->schedule_kind == MP_SCHEDULE_SERIAL && n > 20000)
        return fail(MP_ERR_UNSUPPORTED, "schedule_kind 'serial' is limited to n <= 20000 on the device");
    const int b = cfg->schedule_kind == MP_SCHEDULE_DIAGONAL ? 1 : cfg->tile_b;
    if (b < 1) return fail(MP_ERR_ARG, "tile size must be >= 1, got %d", b);
    if (b > 128 && cfg->schedule_kind != MP_SCHEDULE_SERIAL)
        return fail(MP_ERR_UNSUPPORTED, "tile size %d > 128 is not supported on the device", b);

    int ndev = 0;
    cudaError_t e = cudaGetDeviceCount(&ndev);
    if (e != cudaSuccess || ndev == 0)
        return fail(MP_ERR_CUDA, "no CUDA device available (%s); there is no CPU fallback",
                    cudaGetErrorString(e));
    if (cfg->device < 0 || cfg->device >= ndev)
        return fail(MP_ERR_ARG, "device %d out of range (%d devices)", cfg->device, ndev);
    int cc_major = 0, cc_minor = 0;  // (cudaGetDeviceProperties costs milliseconds)
    CK(cudaDeviceGetAttribute(&cc_major, cudaDevAttrComputeCapabilityMajor, cfg->device));
    CK(cudaDeviceGetAttribute(&cc_minor, cudaDevAttrComputeCapabilityMinor, cfg->device));
    if (cc_major != 10)
        return fail(MP_ERR_CUDA, "device %d is sm_%d%d; this build targets sm_100a", cfg->device,
                    cc_major, cc_minor);

    mp_handle *h = new mp_handle();
    h->dev = cfg->device;
    auto bail = [&](int rc) {
        delete h;
        return rc;
    };
    if (cudaSetDevice(h->dev) != cudaSuccess) return bail(fail(MP_ERR_CUDA, "cudaSetDevice"));
    if (cudaStreamCreateWithFlags(&h->st, cudaStreamNonBlocking) != cudaSuccess)
        return bail(fail(MP_ERR_CUDA, "stream create"));
    tst = h->st;
    tmark("device+stream");
    h->n = n;
    h->m = pair_count(n);
    h->ld = (n + 31) / 32 * 32;
    h->b = b;
    h->kind = cfg->schedule_kind;
    h->flags = cfg->flags;
    h->eps = inst->epsilon;
    const int64_t m = h->m;
    // fast exact division by eps (div_rn) unless eps's significand is all ones
    {
        uint64_t bits;
        std::memcpy(&bits, &h->eps, sizeof(bits));
        const bool all_ones = (bits & 0xFFFFFFFFFFFFFull) == 0xFFFFFFFFFFFFFull;
        h->kc.eps = h->eps;
        const bool in_range = h->eps >= 0x1p-60 && h->eps <= 0x1p+60;  // see div_rn
        h->kc.reps = (all_ones || !in_range || knob("MP_NO_FASTDIV")) ? 0.0 : 1.0 / h->eps;
        h->kc.r3 = 1.0 / 3.0;
    }

    // Host scans of the instance (three passes over C(n,2) doubles: 8 ms each at
    // n = 4000 on one thread) run on all host threads, by ranges of rows.
    const unsigned scan_threads = m > (1 << 20) ? std::max(1u, std::min(16u, std::thread::hardware_concurrency())) : 1u;
    auto scan_rows = [&](auto &&body) {  // body(thread, first row, end row)
        std::vector<std::thread> pool;
        // rows of equal pair count: row i holds n-1-i pairs, so split the pair range evenly
        std::vector<int64_t> cut(scan_threads + 1, n);
        cut[0] = 0;
        for (unsigned q = 1; q < scan_threads; ++q) {
            const double frac = (double)q / scan_threads;
            cut[q] = (int64_t)((double)n * (1.0 - std::sqrt(1.0 - frac)));
        }
        for (unsigned q = 1; q < scan_threads; ++q) pool.emplace_back(body, q, cut[q], cut[q + 1]);
        body(0u, cut[0], cut[1]);
        for (auto &th : pool) th.join();
    };
    auto row_start = [&](int64_t i) { return i * (2 * n - i - 1) / 2; };  // packed index of (i, i+1)

    // regularizer checks (core.py:135-140)
    for (int which = 0; which < 2; ++which) {
        const double *reg = which ? inst->reg_f : inst->reg_x;
        if (!reg) continue;
        std::atomic<int> bad{0}, nonunit{0};
        scan_rows([&](unsigned, int64_t i0, int64_t i1) {
            int b_ = 0, nu = 0;
            for (int64_t p = row_start(i0); p < row_start(i1); ++p) {
                b_ |= !(reg[p] > 0.0);
                nu |= reg[p] != 1.0;
            }
            if (b_) bad = 1;
            if (nu) nonunit = 1;
        });
        if (bad) return bail(fail(MP_ERR_ARG, "regularization weights must be positive"));
        if (nonunit) (which ? h->unit_f : h->unit_x) = false;
    }

    // ---- hub factor of the instance (plan_rounds) ------------------------------
    if (h->kind != MP_SCHEDULE_SERIAL) {
        std::vector<std::vector<int32_t>> part(scan_threads, std::vector<int32_t>((size_t)n, 0));
        scan_rows([&](unsigned q, int64_t i0, int64_t i1) {
            std::vector<int32_t> &dg = part[q];
            int64_t p = row_start(i0);
            for (int64_t i = i0; i < i1; ++i)
                for (int64_t j = i + 1; j < n; ++j, ++p)
                    if (inst->d_flat[p] < 0.5) {
                        ++dg[(size_t)i];
                        ++dg[(size_t)j];
                    }
        });
        std::vector<int32_t> deg((size_t)n, 0);
        for (const auto &dg : part)
            for (int64_t i = 0; i < n; ++i) deg[(size_t)i] += dg[(size_t)i];
        int64_t sum = 0;
        int32_t mx = 0;
        for (int32_t v : deg) sum += v, mx = std::max(mx, v);
        const double mean = (double)sum / (double)n;
        h->hub = mx / std::max(mean, 1.0);
        h->deg = deg;
        if (getenv("MP_VERBOSE")) fprintf(stderr, "[mp] hub factor %.1f (max degree %d, mean %.1f)\n", h->hub, mx, mean);
    }

    // ---- schedule (schedule.tiled_rounds, schedule.py:117-153) -------------
    h->nib = (n + b - 1) / b + 2;
    h->nkb = (n - 1) / b + 2;
    h->tile_of_blk.assign((size_t)(h->nib * h->nkb), -1);
    auto emit = [&](int64_t x, int64_t z) {
        h->round_off.push_back((int64_t)h->tiles.size());
        int64_t cnt = 0;
        for (int64_t c = 0; std::max<int64_t>(x + c * b, 0) + 2 <= z - c * b; ++c) {
            const int64_t tx = x + c * b, tz = z - c * b;
            TileDesc t = make_tile(tx, tz, b);
            const int64_t iblk = (t.ilo + b - 1) / b, kblk = (n - 1 - tz) / b;
            h->tile_of_blk[(size_t)(iblk * h->nkb + kblk)] = (int32_t)h->tiles.size();
            h->tiles.push_back(t);
            h->tile_x.push_back(tx);
            h->tile_round.push_back((int32_t)h->round_cnt.size());
            ++cnt;
        }
        h->round_cnt.push_back(cnt);
    };
    if (h->kind != MP_SCHEDULE_SERIAL) {
        for (int64_t z = n - 1; z >= 2; z -= b) emit(1 - b, z);
        for (int64_t x = 1; x + 2 <= n - 1; x += b) emit(x, n - 1);
    }
    // Launch shape per round and dual-stream numbering (plan_rounds)
    if (h->kind != MP_SCHEDULE_SERIAL) {
        const auto tp0 = std::chrono::steady_clock::now();
        const int rc0 = plan_rounds(h, h->round_cnt);
        if (getenv("MP_VERBOSE"))
            fprintf(stderr, "[mp] plan_rounds %.3f s\n",
                    std::chrono::duration<double>(std::chrono::steady_clock::now() - tp0).count());
        if (rc0) return bail(rc0);
    }
    if (h->kind == MP_SCHEDULE_SERIAL) {
        // cube wavefront: cube levels s = I+J+K, I <= J <= K (mp_cube.cuh)
        const int64_t nb = (n + CUBE_C - 1) / CUBE_C;
        h->nb_cube = nb;
        for (int64_t sl = 0; sl <= 3 * (nb - 1); ++sl) {
            h->cube_off.push_back((int64_t)h->cubes.size());
            int64_t cnt = 0;
            for (int64_t I = 0; I < nb && 3 * I <= sl; ++I)
                for (int64_t J = I; J < nb && I + 2 * J <= sl; ++J) {
                    const int64_t K = sl - I - J;
                    if (K < J || K >= nb) continue;
                    CubeDesc cd{};
                    cd.I = (int32_t)I;
                    cd.J = (int32_t)J;
                    cd.K = (int32_t)K;
                    cd.stream0 = (int64_t)h->cubes.size() * CUBE_WARPS;
                    h->cubes.push_back(cd);
                    ++cnt;
                }
            h->cube_cnt.push_back(cnt);
        }
        h->nstreams = (int64_t)h->cubes.size() * CUBE_WARPS;
    }

    tmark("schedule");
    int rc;
#define TRY(call)                        \
    do {                                 \
        cudaError_t e_ = (call);         \
        if (e_ != cudaSuccess) {         \
            fail(e_ == cudaErrorMemoryAllocation ? MP_ERR_OOM : MP_ERR_CUDA, "%s: %s", #call, \
                 cudaGetErrorString(e_)); \
            return bail(e_ == cudaErrorMemoryAllocation ? MP_ERR_OOM : MP_ERR_CUDA); \
        }                                \
    } while (0)
    TRY(cudaMalloc(&h->d_tiles, std::max<size_t>(h->tiles.size(), 1) * sizeof(TileDesc)));
    TRY(cudaMemcpyAsync(h->d_tiles, h->tiles.data(), h->tiles.size() * sizeof(TileDesc),
                        cudaMemcpyHostToDevice, h->st));
    if (!h->cubes.empty()) {
        TRY(cudaMalloc(&h->d_cubes, h->cubes.size() * sizeof(CubeDesc)));
        TRY(cudaMemcpyAsync(h->d_cubes, h->cubes.data(), h->cubes.size() * sizeof(CubeDesc),
                            cudaMemcpyHostToDevice, h->st));
    }

    // ---- instance and state --------------------------------------------------
    const size_t dense = (size_t)n * h->ld * sizeof(double);
    TRY(cudaMalloc(&h->x, dense));
    TRY(cudaMemsetAsync(h->x, 0, dense, h->st));  // x = 0 (solver.py:112)
    TRY(cudaMalloc(&h->snap_x, dense));
    const auto tm0 = std::chrono::steady_clock::now();
    if ((rc = make_x_tmap(h))) return bail(rc);
    if (getenv("MP_VERBOSE"))
        fprintf(stderr, "[mp] make_x_tmap %.3f s\n",
                std::chrono::duration<double>(std::chrono::steady_clock::now() - tm0).count());
    h->tma_store = knob("MP_NO_TMA_STORE") ? 0 : 1;
    tmark("x+tmap");
    TRY(cudaMalloc(&h->tmp, m * sizeof(double)));
    if ((rc = upload_packed(h, &h->d, inst->d_flat))) return bail(rc);
    if ((rc = upload_packed(h, &h->w, inst->w_flat))) return bail(rc);
    const int egrid = grid_for(m, 256, 148 * 16);
    if (!h->unit_x) {
        if ((rc = upload_packed(h, &h->regx, inst->reg_x))) return bail(rc);
        TRY(cudaMalloc(&h->winvx, dense));
        reciprocal_kernel<<<egrid, 256, 0, h->st>>>(h->regx, h->tmp, m);  // solver.py:173
        expand_kernel<<<egrid, 256, 0, h->st>>>(h->tmp, h->winvx, h->ld, n, m);
        TRY(cudaGetLastError());
    }
    if (!h->unit_f) {
        if ((rc = upload_packed(h, &h->regf, inst->reg_f))) return bail(rc);
        TRY(cudaMalloc(&h->winvf, m * sizeof(double)));
        reciprocal_kernel<<<egrid, 256, 0, h->st>>>(h->regf, h->winvf, m);  // solver.py:174
        TRY(cudaGetLastError());
    }
    // f = -w / (eps * reg_f)  (solver.py:112), computed as numpy does
    // f = -w / (eps * reg_f) (solver.py:108-113), IEEE division on the device
    TRY(cudaMalloc(&h->f, m * sizeof(double)));
    f_init_kernel<<<egrid, 256, 0, h->st>>>(h->w, h->unit_f ? nullptr : h->regf, h->eps, h->f, m);
    TRY(cudaGetLastError());
    tmark("upload d,w,f");
    TRY(cudaMalloc(&h->pu, m * sizeof(double)));
    TRY(cudaMalloc(&h->pl, m * sizeof(double)));
    TRY(cudaMemsetAsync(h->pu, 0, m * sizeof(double), h->st));
    TRY(cudaMemsetAsync(h->pl, 0, m * sizeof(double), h->st));
    TRY(cudaMalloc(&h->snap_f, m * sizeof(double)));
    TRY(cudaMalloc(&h->snap_pu, m * sizeof(double)));
    TRY(cudaMalloc(&h->snap_pl, m * sizeof(double)));

    // ---- duals and bookkeeping -------------------------------------------------
    // about one chunk per stream: the first pass writes into most streams
    int32_t cap0 = (int32_t)std::min<int64_t>(std::max<int64_t>(4096, h->nstreams + h->nstreams / 4), 1 << 22);
    if (const char *e = knob("MP_POOL_CAP0")) cap0 = std::max(1, atoi(e));  // tests: force overflow
    if (!knob("MP_POOL_CAP0")) {
        std::lock_guard<std::mutex> lk(g_hint_mu);
        auto it = g_pool_hint.find({n, b, h->kind, h->nstreams});
        if (it != g_pool_hint.end()) cap0 = std::max(cap0, it->second);
    }
    if ((rc = alloc_pool(h, 0, cap0))) return bail(rc);
    if ((rc = alloc_pool(h, 1, cap0))) return bail(rc);
    h->pair_grid = grid_for(m, 256, 148 * 8);
    TRY(cudaMalloc(&h->partials, (size_t)h->pair_grid * 4 * sizeof(double)));
    TRY(cudaMalloc(&h->ctr, sizeof(PassCounters)));
    TRY(cudaMalloc(&h->d_stats, sizeof(DevStats)));
    TRY(cudaMalloc(&h->d_scan, sizeof(unsigned long long)));
    TRY(pin_malloc(reinterpret_cast<void **>(&h->h_stats), sizeof(DevStats)));
    for (auto &ev : h->ev) TRY(cudaEventCreate(&ev));
    TRY(cudaStreamSynchronize(h->st));
    tmark("pools+rest");
#undef TRY
    *out = h;
    return MP_OK;
}

void mp_destroy(mp_handle *h) { delete h; }

}  // extern "C"

namespace {

// Kernels one session launches per pass (its own, not library calls).
int64_t launches_per_pass(const mp_handle *h) {
    int64_t c = 2;  // pair phase + finalize
    for (size_t r = 0; r < h->round_cnt.size(); ++r) {
        if (h->df_on && r > h->df_r0) continue;  // one dataflow launch for the second family
        c += (h->sh.on ? h->sh.my_cnt[r] : h->round_cnt[r]) ? 1 : 0;
        if (round_exchanges(h, r)) c += (h->sh.sp_cnt[r] > 0) + (h->sh.rp_cnt[r] > 0);  // pack, unpack
    }
    if (h->kind == MP_SCHEDULE_SERIAL)
        for (int64_t cnt : h->cube_cnt) c += cnt ? 1 : 0;
    if (h->sh.on && h->sh.local && h->sh.world > 1 && h->sh.rank == 0) c += 1;  // counter reduce
    return c;
}

// run_pass x npasses (solver.py:166-210) for a group of sessions solving one
// instance together (see enqueue_group_pass); stats come from hs[0].
int run_group(std::vector<mp_handle *> &hs, int32_t npasses, mp_pass_stats *out) {
    mp_handle *h0 = hs[0];
    for (mp_handle *h : hs) {
        h->metric_ms = h->pair_ms = 0.0;
        h->launches = 0;
    }
    PassCounters **d_ctrs = nullptr;
    if (hs.size() > 1) {
        std::vector<PassCounters *> ptrs;
        for (mp_handle *h : hs) ptrs.push_back(h->ctr);
        CK(cudaMalloc(&d_ctrs, ptrs.size() * sizeof(PassCounters *)));
        CK(cudaMemcpy(d_ctrs, ptrs.data(), ptrs.size() * sizeof(PassCounters *), cudaMemcpyHostToDevice));
    }
    struct Free {
        PassCounters **p;
        ~Free() { cudaFree(p); }
    } free_ctrs{d_ctrs};
    auto local_chunks = [](const mp_handle *h) {
        return h->sh.on ? h->sh.h_local->chunks_used : h->h_stats->chunks_used;
    };
    for (int32_t k = 0; k < npasses; ++k) {
        const int wp = h0->rp ^ 1;
        for (mp_handle *h : hs) {
            // keep the write pool comfortably above the last pass's usage
            int64_t want = std::max<int64_t>(h->pool[wp].cap, 2 * (int64_t)h->pool_used[h->rp] + 1024);
            if (want > h->pool[wp].cap) {
                // grow geometrically: a reallocation synchronises and costs ms
                want = std::max<int64_t>(want, (int64_t)h->pool[wp].cap * 3 / 2);
                if (getenv("MP_VERBOSE")) fprintf(stderr, "[mp] pool %d: %d -> %lld chunks\n", wp, h->pool[wp].cap, (long long)want);
                CK(cudaStreamSynchronize(h->st));
                int rc = alloc_pool(h, wp, (int32_t)std::min<int64_t>(want, 0x7fffffff));
                if (rc) return rc;
            }
        }
        for (int attempt = 0;; ++attempt) {
            int rc = enqueue_group_pass(hs, d_ctrs);
            if (rc) return rc;
            for (mp_handle *h : hs) CK(cudaStreamSynchronize(h->st));
            if (!h0->h_stats->overflow) break;  // all-reduced: every rank agrees
            if (getenv("MP_VERBOSE")) fprintf(stderr, "[mp] pass %lld: dual pool overflow, redo\n", (long long)h0->pass_index);
            // dual pool overflow: roll the pass back, grow the pools, redo it
            for (mp_handle *h : hs) {
                rc = restore_snapshot(h);
                if (rc) return rc;
                CK(cudaStreamSynchronize(h->st));
                const int64_t grow = std::max<int64_t>(2 * (int64_t)h->pool[wp].cap,
                                                       (int64_t)local_chunks(h) * 2);
                if (attempt > 8 || grow > 0x7fffffff)
                    return fail(MP_ERR_OOM, "dual pool cannot grow further");
                rc = alloc_pool(h, wp, (int32_t)grow);
                if (rc) return rc;
            }
        }
        for (mp_handle *h : hs) {
            // device time of the pass (snapshot .. finalize), metric vs pair phase
            float ms_metric = 0.f, ms_pair = 0.f;
            CK(cudaEventElapsedTime(&ms_metric, h->ev[1], h->ev[2]));
            CK(cudaEventElapsedTime(&ms_pair, h->ev[2], h->ev[3]));
            h->metric_ms += ms_metric;
            h->pair_ms += ms_pair;
            h->launches += launches_per_pass(h);
            h->pool_used[wp] = local_chunks(h);
            h->rp = wp;
            h->nnz = h->sh.on ? (int64_t)h->sh.h_local->nnz : (int64_t)h->h_stats->nnz;
            h->pass_index++;
        }
        float ms_all = 0.f;
        CK(cudaEventElapsedTime(&ms_all, h0->ev[0], h0->ev[3]));
        const DevStats &s = *h0->h_stats;
        mp_pass_stats &o = out[k];
        o.pass_index = h0->pass_index - 1;
        o.steps = 3 * (h0->n * (h0->n - 1) * (h0->n - 2) / 6) + 2 * h0->m;
        o.nnz_metric = (int64_t)s.nnz;
        o.primal_objective = s.primal;
        o.dual_objective = s.dual;
        o.duality_gap = s.gap;
        o.max_violation = s.viol;
        o.wall_time = ms_all * 1e-3;
        if (s.nonfinite) {
            return fail(MP_ERR_NONFINITE, "non-finite value in state after pass %lld",
                        (long long)o.pass_index);
        }
    }
    return MP_OK;
}

}  // namespace

extern "C" {

int mp_run_passes(mp_handle *h, int32_t npasses, mp_pass_stats *out) {
    g_err.clear();
    if (!h || npasses < 0 || (npasses > 0 && !out)) return fail(MP_ERR_ARG, "bad argument");
    if (h->sh.on && h->sh.local && h->sh.world > 1)
        return fail(MP_ERR_ARG, "a local-transport shard runs only through mp_group_run_passes");
    CK(cudaSetDevice(h->dev));
    std::vector<mp_handle *> hs{h};
    return run_group(hs, npasses, out);
}

int mp_get_state(mp_handle *h, double *xv, double *fv) {
    g_err.clear();
    if (!h) return fail(MP_ERR_ARG, "null handle");
    CK(cudaSetDevice(h->dev));
    const int g = grid_for(h->m, 256, 148 * 16);
    // Straight into the caller's buffers: the driver stages a pageable copy at
    // ~18 GB/s on this host, and what dominates either way is the first touch of
    // the caller's fresh pages; a pinned stage of 2 x 8 m bytes would cost more
    // to allocate (58 ms per 128 MB) than it ever saves here.
    const size_t mb = (size_t)h->m * sizeof(double);
    if (xv) {
        pack_kernel<<<g, 256, 0, h->st>>>(h->x, h->tmp, h->ld, h->n, h->m);
        CK(cudaGetLastError());
    }
    prefault_output(xv, mb);  // (under the pack kernel)
    prefault_output(fv, mb);
    if (xv) CK(cudaMemcpyAsync(xv, h->tmp, mb, cudaMemcpyDeviceToHost, h->st));
    if (fv) CK(cudaMemcpyAsync(fv, h->f, mb, cudaMemcpyDeviceToHost, h->st));
    CK(cudaStreamSynchronize(h->st));
    return MP_OK;
}

int mp_set_state(mp_handle *h, const double *xv, const double *fv) {
    g_err.clear();
    if (!h) return fail(MP_ERR_ARG, "null handle");
    CK(cudaSetDevice(h->dev));
    const int g = grid_for(h->m, 256, 148 * 16);
    if (xv) {
        CK(cudaMemcpyAsync(h->tmp, xv, h->m * sizeof(double), cudaMemcpyHostToDevice, h->st));
        expand_kernel<<<g, 256, 0, h->st>>>(h->tmp, h->x, h->ld, h->n, h->m);
        CK(cudaGetLastError());
    }
    if (fv) CK(cudaMemcpyAsync(h->f, fv, h->m * sizeof(double), cudaMemcpyHostToDevice, h->st));
    CK(cudaStreamSynchronize(h->st));
    return MP_OK;
}

int64_t mp_dual_count(mp_handle *h) { return h ? h->nnz : -1; }

}  // extern "C"

namespace {

// Duals of this session in the reference's single-worker visit order; order[e]
// (optional) = schedule index of the entry's tile, so the shards of a sharded
// solve merge into the global order with a stable sort on it.
int get_duals_impl(mp_handle *h, int64_t *keys, double *vals, double *pair_duals, int64_t *order) {
    g_err.clear();
    if (!h) return fail(MP_ERR_ARG, "null handle");
    CK(cudaSetDevice(h->dev));
    if (pair_duals) {
        // interleaved on the device (the pass-start snapshot of x is free between
        // passes and holds n x ld >= 2 m values), one copy into the caller's array
        interleave2_kernel<<<grid_for(h->m, 256, 148 * 16), 256, 0, h->st>>>(h->pu, h->pl, h->snap_x, h->m);
        CK(cudaGetLastError());
        prefault_output(pair_duals, 2 * (size_t)h->m * sizeof(double));
        CK(cudaMemcpyAsync(pair_duals, h->snap_x, 2 * (size_t)h->m * sizeof(double), cudaMemcpyDeviceToHost, h->st));
        CK(cudaStreamSynchronize(h->st));
    }
    if (!keys && !vals) return MP_OK;
    const DualPool &P = h->pool[h->rp];
    const int64_t used = h->pool_used[h->rp];
    const size_t rec_bytes = (size_t)used * sizeof(ChunkRec);
    // (pageable: pinning a stage of this size costs more than the copy's ~18
    // GB/s loses against a pinned one, and the first call of a process pays it)
    const size_t stg_bytes = rec_bytes + (size_t)std::max<int64_t>(h->nstreams, 1) * sizeof(int32_t);
    std::unique_ptr<char[]> stg_own(new (std::nothrow) char[stg_bytes]);
    char *stg = stg_own.get();
    if (!stg) return fail(MP_ERR_OOM, "dual export buffer");
    prefault_output(stg, stg_bytes);
    const ChunkRec *hr = reinterpret_cast<const ChunkRec *>(stg);
    const int32_t *hh = reinterpret_cast<const int32_t *>(stg + rec_bytes);
    if (used)
        CK(cudaMemcpyAsync(stg, P.rec, rec_bytes, cudaMemcpyDeviceToHost, h->st));
    if (h->nstreams)
        CK(cudaMemcpyAsync(stg + rec_bytes, P.head, (size_t)h->nstreams * sizeof(int32_t),
                           cudaMemcpyDeviceToHost, h->st));
    CK(cudaStreamSynchronize(h->st));
    const int64_t n = h->n;
    int64_t outpos = 0;
    struct E {
        int64_t rank[5];
        int64_t key;
        double val;
    };
    if (h->kind == MP_SCHEDULE_SERIAL) {
        // serial visit order is lexicographic (i, j, k, kind) = ascending key code
        std::vector<std::pair<int64_t, double>> all;
        constexpr int c = CUBE_C, S = CUBE_S;
        for (int64_t s = 0; s < h->nstreams; ++s) {
            const CubeDesc &cd = h->cubes[(size_t)(s / CUBE_WARPS)];
            const int64_t warp = s % CUBE_WARPS, Lmin = (int64_t)(cd.I + cd.J + cd.K) * c;
            int32_t ch = used ? hh[(size_t)s] : -1;
            while (ch >= 0 && ch < used) {
                for (int e = 0; e < CHUNK; ++e) {
                    const uint32_t key = hr[(size_t)ch].keys[e];
                    if (key == KEY_END) break;
                    const int64_t lvl = key / (S * 96), rem = key % (S * 96);
                    const int64_t sl = rem / 96, lane = (rem % 96) / 3, kind = rem % 3;
                    const int64_t q = (warp * S + sl) * 32 + lane;
                    const int64_t i = (int64_t)cd.I * c + q / c, k = (int64_t)cd.K * c + q % c;
                    const int64_t j = Lmin + lvl - i - k;
                    all.push_back({((i * n + j) * n + k) * 3 + kind, hr[(size_t)ch].vals[e]});
                }
                ch = hr[(size_t)ch].next;
            }
        }
        std::sort(all.begin(), all.end());
        if ((int64_t)all.size() != h->nnz)
            return fail(MP_ERR_CUDA, "dual store inconsistent: %lld vs %lld", (long long)all.size(),
                        (long long)h->nnz);
        for (size_t e = 0; e < all.size(); ++e) {
            if (keys) keys[e] = all[e].first;
            if (vals) vals[e] = all[e].second;
            if (order) order[e] = (int64_t)e;
        }
        return MP_OK;
    }
    // Tiles are independent: count each tile's entries (walk its streams'
    // chunk chains), prefix-sum the counts into output offsets, then decode,
    // order and write the tiles on all host threads.
    const size_t nt = h->tiles.size();
    auto tile_streams = [&](size_t t) {
        const mp_handle::RoundCfg &rc = h->rcfg[(size_t)h->tile_round[t]];
        return rc.C * rc.NWC;
    };
    std::vector<int64_t> toff(nt + 1, 0);
    const unsigned hw = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
    const unsigned nthreads = used > 4096 ? hw : 1u;
    auto parallel_tiles = [&](auto &&body) {
        std::atomic<size_t> next{0};
        auto work = [&] {
            for (;;) {
                const size_t t0 = next.fetch_add(64);
                if (t0 >= nt) break;
                for (size_t t = t0; t < std::min(nt, t0 + 64); ++t) body(t);
            }
        };
        std::vector<std::thread> pool;
        for (unsigned q = 1; q < nthreads; ++q) pool.emplace_back(work);
        work();
        for (auto &th : pool) th.join();
    };
    parallel_tiles([&](size_t t) {
        int64_t cnt = 0;
        for (int w = 0; w < tile_streams(t); ++w) {
            int32_t c = used ? hh[(size_t)(h->tiles[t].stream0 + w)] : -1;
            while (c >= 0 && c < used) {
                int e = 0;
                while (e < CHUNK && hr[(size_t)c].keys[e] != KEY_END) ++e;
                cnt += e;
                c = hr[(size_t)c].next;
            }
        }
        toff[t + 1] = cnt;
    });
    for (size_t t = 0; t < nt; ++t) toff[t + 1] += toff[t];
    outpos = toff[nt];
    if (outpos != h->nnz) return fail(MP_ERR_CUDA, "dual store inconsistent: %lld vs %lld",
                                      (long long)outpos, (long long)h->nnz);
    parallel_tiles([&](size_t t) {
        if (toff[t + 1] == toff[t]) return;
        std::vector<E> te;
        te.reserve((size_t)(toff[t + 1] - toff[t]));
        const int64_t tx = h->tile_x[t];
        for (int w = 0; w < tile_streams(t); ++w) {
            int32_t c = hh[(size_t)(h->tiles[t].stream0 + w)];
            while (c >= 0 && c < used) {
                for (int e = 0; e < CHUNK; ++e) {
                    const uint32_t key = hr[(size_t)c].keys[e];
                    if (key == KEY_END) break;
                    Decoded dd = decode_entry(h, (int64_t)t, w, key);
                    E en;
                    // reference cube order inside a tile (_kernels.py:81-97)
                    en.rank[0] = (dd.j - (tx + 1)) / h->b;
                    en.rank[1] = dd.k;
                    en.rank[2] = dd.j;
                    en.rank[3] = dd.i;
                    en.rank[4] = dd.kind;
                    en.key = ((dd.i * n + dd.j) * n + dd.k) * 3 + dd.kind;
                    en.val = hr[(size_t)c].vals[e];
                    te.push_back(en);
                }
                c = hr[(size_t)c].next;
            }
        }
        std::sort(te.begin(), te.end(), [](const E &a, const E &b) {
            return std::lexicographical_compare(a.rank, a.rank + 5, b.rank, b.rank + 5);
        });
        int64_t o = toff[t];
        for (const E &en : te) {
            if (keys) keys[o] = en.key;
            if (vals) vals[o] = en.val;
            if (order) order[o] = (int64_t)t;
            ++o;
        }
    });
    if (outpos != h->nnz) return fail(MP_ERR_CUDA, "dual store inconsistent: %lld vs %lld",
                                      (long long)outpos, (long long)h->nnz);
    return MP_OK;
}

}  // namespace

extern "C" {

int mp_get_duals(mp_handle *h, int64_t *keys, double *vals, double *pair_duals) {
    return get_duals_impl(h, keys, vals, pair_duals, nullptr);
}

int mp_get_duals_ranked(mp_handle *h, int64_t *keys, double *vals, int64_t *order) {
    return get_duals_impl(h, keys, vals, nullptr, order);
}

int mp_set_duals(mp_handle *h, int64_t nnz, const int64_t *keys, const double *vals,
                 const double *pair_duals) {
    g_err.clear();
    if (!h || nnz < 0 || (nnz > 0 && (!keys || !vals))) return fail(MP_ERR_ARG, "bad argument");
    CK(cudaSetDevice(h->dev));
    const int64_t n = h->n, b = h->b;
    // bucket entries by warp stream
    std::vector<std::pair<int64_t, std::pair<uint32_t, double>>> ents;
    ents.reserve((size_t)nnz);
    for (int64_t e = 0; e < nnz; ++e) {
        const int64_t code = keys[e];
        if (code < 0) return fail(MP_ERR_ARG, "negative dual key");
        const int64_t kind = code % 3, t3 = code / 3;
        const int64_t k = t3 % n, j = (t3 / n) % n, i = t3 / (n * n);
        if (!(i < j && j < k && k < n)) return fail(MP_ERR_ARG, "invalid metric key %lld", (long long)code);
        if (!(vals[e] > 0.0) || !std::isfinite(vals[e]))
            return fail(MP_ERR_ARG, "dual values must be positive and finite");
        if (h->kind == MP_SCHEDULE_SERIAL) {
            constexpr int c = CUBE_C, S = CUBE_S;
            const int64_t I = i / c, J = j / c, K = k / c;
            const int64_t ci = cube_index(h, I, J, K);
            const int64_t q = (i - I * c) * c + (k - K * c);
            const int64_t warp = q / (32 * S), sl = (q / 32) % S, lane = q % 32;
            const int64_t lvl = i + j + k - (I + J + K) * c;
            ents.push_back({h->cubes[(size_t)ci].stream0 + warp,
                            {(uint32_t)((lvl * S + sl) * 96 + lane * 3 + kind), vals[e]}});
            continue;
        }
        const int64_t iblk = (i + b - 1) / b, kblk = (n - 1 - k) / b;
        if (iblk >= h->nib || kblk >= h->nkb) return fail(MP_ERR_ARG, "key outside schedule");
        const int32_t t = h->tile_of_blk[(size_t)(iblk * h->nkb + kblk)];
        if (t < 0) return fail(MP_ERR_ARG, "key outside schedule");
        if (h->sh.on && h->sh.owner[(size_t)t] != h->sh.rank) continue;  // another shard's dual
        const TileDesc &T = h->tiles[(size_t)t];
        const mp_handle::RoundCfg &c = h->rcfg[(size_t)h->tile_round[(size_t)t]];
        int64_t band = 0;
        while (band + 1 < c.C && c.bst[(size_t)band + 1] <= i - T.ilo) ++band;
        const int64_t S = c.S;
        const int64_t nrows = (int64_t)T.ihi - T.ilo + 1;
        const int64_t r0 = c.bst[(size_t)band], r1 = std::min<int64_t>(b, c.bst[(size_t)band + 1]),
                      rbc = std::max<int64_t>(1, std::min<int64_t>(r1, nrows) - r0);
        const int64_t q = c.colm ? (k - T.klo) * rbc + (i - T.ilo - r0) : (i - T.ilo - r0) * b + (k - T.klo);
        const int64_t LW = band_lanes(c.blw[(size_t)band], c.NWC, c.S, (int)rbc, (int)(r1 - r0), (int)b, c.colm);
        const int64_t w = q / (LW * S), s = (q % (LW * S)) / LW, lane = q % LW;
        const int64_t lvl = i + j + k - T.Lbeg;
        const uint32_t key32 = (uint32_t)(((lvl * S + s) * 96) + lane * 3 + kind);
        ents.push_back({T.stream0 + band * c.NWC + w, {key32, vals[e]}});
    }
    std::sort(ents.begin(), ents.end(), [](const auto &a, const auto &c) {
        return a.first != c.first ? a.first < c.first : a.second.first < c.second.first;
    });
    for (size_t e = 1; e < ents.size(); ++e)
        if (ents[e].first == ents[e - 1].first && ents[e].second.first == ents[e - 1].second.first)
            return fail(MP_ERR_ARG, "duplicate dual key");
    // pack into chunk records
    std::vector<ChunkRec> hr;
    std::vector<int32_t> hh((size_t)h->nstreams, -1);
    size_t e = 0;
    while (e < ents.size()) {
        const int64_t s = ents[e].first;
        int32_t prev = -1;
        size_t cnt = 0;
        while (e < ents.size() && ents[e].first == s) {
            if (cnt % CHUNK == 0) {
                const int32_t c = (int32_t)hr.size();
                ChunkRec r;
                std::memset(&r, 0, sizeof(r));
                for (int q = 0; q < CHUNK; ++q) r.keys[q] = KEY_END;
                r.next = -1;
                hr.push_back(r);
                if (prev >= 0) hr[(size_t)prev].next = c;
                else hh[(size_t)s] = c;
                prev = c;
            }
            hr[(size_t)prev].keys[cnt % CHUNK] = ents[e].second.first;
            hr[(size_t)prev].vals[cnt % CHUNK] = ents[e].second.second;
            ++cnt;
            ++e;
        }
    }
    const int32_t used = (int32_t)hr.size();
    const int rp = h->rp;
    if (used > h->pool[rp].cap) {
        int rc = alloc_pool(h, rp, std::max<int32_t>(used * 2, 4096));
        if (rc) return rc;
    }
    DualPool &P = h->pool[rp];
    if (used)
        CK(cudaMemcpyAsync(P.rec, hr.data(), hr.size() * sizeof(ChunkRec), cudaMemcpyHostToDevice, h->st));
    if (h->nstreams)
        CK(cudaMemcpyAsync(P.head, hh.data(), hh.size() * sizeof(int32_t), cudaMemcpyHostToDevice, h->st));
    CK(cudaStreamSynchronize(h->st));
    h->pool_used[rp] = used;
    h->nnz = (int64_t)ents.size();
    if (pair_duals) {
        std::vector<double> a((size_t)h->m), c((size_t)h->m);
        for (int64_t p = 0; p < h->m; ++p) {
            a[(size_t)p] = pair_duals[2 * p];
            c[(size_t)p] = pair_duals[2 * p + 1];
        }
        CK(cudaMemcpyAsync(h->pu, a.data(), h->m * sizeof(double), cudaMemcpyHostToDevice, h->st));
        CK(cudaMemcpyAsync(h->pl, c.data(), h->m * sizeof(double), cudaMemcpyHostToDevice, h->st));
        CK(cudaStreamSynchronize(h->st));
    }
    CK(cudaStreamSynchronize(h->st));
    return MP_OK;
}

int mp_state_max_violation(mp_handle *h, double *out) {
    g_err.clear();
    if (!h || !out) return fail(MP_ERR_ARG, "bad argument");
    CK(cudaSetDevice(h->dev));
    CK(cudaMemsetAsync(h->d_scan, 0, sizeof(unsigned long long), h->st));
    scan_metric_kernel<<<(unsigned)std::max<int64_t>(h->n - 2, 1), 256, 0, h->st>>>(h->x, h->ld, h->n, h->d_scan);
    CK(cudaGetLastError());
    scan_pair_kernel<<<grid_for(h->m, 256, 148 * 16), 256, 0, h->st>>>(h->x, h->ld, h->f, h->d, h->n,
                                                                        h->m, h->d_scan);
    CK(cudaGetLastError());
    unsigned long long bits = 0;
    CK(cudaMemcpyAsync(&bits, h->d_scan, sizeof(bits), cudaMemcpyDeviceToHost, h->st));
    CK(cudaStreamSynchronize(h->st));
    double v;
    std::memcpy(&v, &bits, sizeof(v));
    *out = v;
    return MP_OK;
}

int mp_get_timing(mp_handle *h, double *metric_ms, double *pair_ms, int64_t *launches) {
    if (!h) return fail(MP_ERR_ARG, "null handle");
    if (metric_ms) *metric_ms = h->metric_ms;
    if (pair_ms) *pair_ms = h->pair_ms;
    if (launches) *launches = h->launches;
    return MP_OK;
}

int mp_trace(mp_handle *h, int32_t enable, uint64_t *out, int32_t nslots) {
    g_err.clear();
    if (!h) return fail(MP_ERR_ARG, "null handle");
    CK(cudaSetDevice(h->dev));
#if defined(MP_TILETIME)
    const size_t ns = TT_SLOTS;  // diagnostic build: per-tile times
#elif defined(MP_TIMELINE)
    const size_t ns = TL_SLOTS;  // diagnostic build: the per-batch timeline
#else
    const size_t ns = TR_NSLOTS;
#endif
    if (enable && !h->trace) {
        CK(cudaMalloc(&h->trace, ns * sizeof(unsigned long long)));
        CK(cudaMemsetAsync(h->trace, 0, ns * sizeof(unsigned long long), h->st));
    }
    if (out && h->trace) {
        std::vector<unsigned long long> buf(ns);
        CK(cudaMemcpyAsync(buf.data(), h->trace, ns * sizeof(unsigned long long), cudaMemcpyDeviceToHost, h->st));
        CK(cudaStreamSynchronize(h->st));
        for (size_t i = 0; i < (size_t)nslots && i < ns; ++i) out[i] = buf[i];
        CK(cudaMemsetAsync(h->trace, 0, ns * sizeof(unsigned long long), h->st));
    }
    if (!enable && h->trace) {
        CK(cudaStreamSynchronize(h->st));
        cudaFree(h->trace);
        h->trace = nullptr;
    }
    return MP_OK;
}

int mp_flush_l2(mp_handle *h) {
    g_err.clear();
    if (!h) return fail(MP_ERR_ARG, "null handle");
    CK(cudaSetDevice(h->dev));
    if (!h->flush) {
        h->flush_bytes = (size_t)256 << 20;
        CK(cudaMalloc(&h->flush, h->flush_bytes));
    }
    static unsigned char v = 0;
    CK(cudaMemsetAsync(h->flush, ++v, h->flush_bytes, h->st));
    CK(cudaStreamSynchronize(h->st));
    return MP_OK;
}

// ---- sharded execution (mp_shard.cuh) -----------------------

int mp_shard_plan(int64_t n, int32_t b, int32_t world, int32_t *owner, int64_t *ntiles) {
    g_err.clear();
    if (n < 3 || b < 1 || world < 1 || !ntiles) return fail(MP_ERR_ARG, "bad argument");
    std::vector<int64_t> tx, tz, rc;
    enumerate_tiles(n, b, tx, tz, rc);
    *ntiles = (int64_t)tx.size();
    if (owner) {
        std::vector<int32_t> o;
        lpt_owner(b, world, tx, tz, rc, o);
        std::copy(o.begin(), o.end(), owner);
    }
    return MP_OK;
}

int mp_nccl_unique_id(void *id) {
    g_err.clear();
    if (!id) return fail(MP_ERR_ARG, "null argument");
    const NcclApi &N = nccl_api();
    if (!N.getUniqueId) return fail(MP_ERR_UNSUPPORTED, "NCCL unavailable: %s", N.why.c_str());
    ncclUniqueId u;
    NCK(N.getUniqueId(&u));
    std::memcpy(id, &u, sizeof(u));
    return MP_OK;
}

}  // extern "C"

namespace {

// Re-plan the launch shapes for `cnt_r` tiles per round and renumber the dual
// streams (tile descriptors and stream heads on the device follow).
int replan(mp_handle *h, const std::vector<int64_t> &cnt_r) {
    int rc = plan_rounds(h, cnt_r);
    if (rc) return rc;
    CK(cudaMemcpy(h->d_tiles, h->tiles.data(), h->tiles.size() * sizeof(TileDesc), cudaMemcpyHostToDevice));
    for (auto &p : h->pool) {  // stream heads for the new numbering
        cudaFree(p.head);
        p.head = nullptr;
        CK(cudaMalloc(&p.head, (size_t)std::max<int64_t>(h->nstreams, 1) * sizeof(int32_t)));
        CK(cudaMemset(p.head, 0xff, (size_t)std::max<int64_t>(h->nstreams, 1) * sizeof(int32_t)));
    }
    return MP_OK;
}

// The exchange plan of rank `rank` (mp_shard.cuh): for every tile of every
// round, in schedule order, the blocks of its footprint with the rank of each
// block's next toucher; runs of blocks with one destination become pieces.
// Every rank enumerates all tiles, so both ends of a (source, destination)
// pair lay the pieces out alike.
struct ExchangePlan {
    std::vector<PieceDesc> send, recv;
    std::vector<int64_t> sp_off, sp_cnt, rp_off, rp_cnt, scnt, soff, rcnt, roff;
    std::vector<char> round_any;
    std::vector<int64_t> pairs;  // per round x source x destination: pairs sent (no padding)
    int64_t send_max = 0, recv_max = 0, sent = 0, received = 0;
};

void plan_exchange(const mp_handle *h, const std::vector<int32_t> &owner, int world, int rank,
                   ExchangePlan &P) {
    const int64_t n = h->n, b = h->b, nkb = h->nkb, nib = h->nib;
    const size_t R = h->round_cnt.size();
    auto tile_at = [&](int64_t I, int64_t K) -> int32_t {
        return (I < 0 || K < 0 || I >= nib || K >= nkb) ? -1 : h->tile_of_blk[(size_t)(I * nkb + K)];
    };
    auto exists = [&](int64_t I, int64_t K) { return tile_at(I, K) >= 0; };
    auto row_block = [&](int64_t r) { return r <= 0 ? (int64_t)0 : (r + b - 1) / b; };
    auto col_block = [&](int64_t c) { return (n - 1 - c) / b; };
    P.scnt.assign(R * world, 0);
    P.rcnt.assign(R * world, 0);
    P.soff.assign(R * world, 0);
    P.roff.assign(R * world, 0);
    P.round_any.assign(R, 0);
    P.pairs.assign(R * world * world, 0);
    std::vector<std::vector<PieceDesc>> sp((size_t)world), rp((size_t)world);  // this round, per peer
    std::vector<int64_t> cnt((size_t)world * world);                          // this round, src x dst
    for (size_t r = 0; r < R; ++r) {
        for (auto &v : sp) v.clear();
        for (auto &v : rp) v.clear();
        std::fill(cnt.begin(), cnt.end(), 0);
        // rectangle rows [r0, r1] x columns [c0, c1] from `src` to `dst` (-1: every other rank)
        auto add = [&](int src, int dst, int64_t r0, int64_t r1, int64_t c0, int64_t c1) {
            if (r1 < r0 || c1 < c0) return;
            int64_t valid = 0;  // pairs row < col of the rectangle
            for (int64_t q = r0; q <= r1; ++q) valid += std::max<int64_t>(0, c1 - std::max(c0, q + 1) + 1);
            for (int d = 0; d < world; ++d) {
                if (d == src || (dst >= 0 && d != dst)) continue;
                P.pairs[(r * world + src) * world + d] += valid;
                int64_t &off = cnt[(size_t)src * world + d];
                const int64_t nr = r1 - r0 + 1, nc = c1 - c0 + 1;
                // split into pieces of at most PIECE_MAX values along the longer side
                const int64_t rh = nc >= nr ? nr : std::max<int64_t>(1, PIECE_MAX / nc);
                const int64_t cw = nc >= nr ? std::max<int64_t>(1, PIECE_MAX / nr) : nc;
                for (int64_t a = 0; a < nr; a += rh)
                    for (int64_t c = 0; c < nc; c += cw) {
                        PieceDesc pc;
                        pc.row0 = (int32_t)(r0 + a);
                        pc.nrows = (int32_t)std::min(rh, nr - a);
                        pc.col0 = (int32_t)(c0 + c);
                        pc.ncols = (int32_t)std::min(cw, nc - c);
                        pc.off = off;
                        off += (int64_t)pc.nrows * pc.ncols;
                        if (src == rank) sp[(size_t)d].push_back(pc);
                        if (d == rank) rp[(size_t)src].push_back(pc);
                    }
            }
        };
        for (int64_t t = h->round_off[r]; t < h->round_off[r] + h->round_cnt[r]; ++t) {
            const TileDesc &T = h->tiles[(size_t)t];
            const int64_t I = row_block(T.ilo), K = col_block(T.z);
            const int src = owner[(size_t)t];
            auto dest = [&](int64_t Ia, int64_t Kb) {  // rank of the block's next toucher, -1: all
                int64_t nI, nK;
                if (!next_toucher(Ia, Kb, I, K, exists, nI, nK)) return -1;
                return (int)owner[(size_t)tile_at(nI, nK)];
            };
            add(src, dest(I, K), T.ilo, T.ihi, T.klo, T.z);  // RK
            // WR: rows R x columns [wr0, wr1], by column block from the lowest columns up
            const int64_t wr0 = std::max<int64_t>(T.jlo, T.ilo + 1), wr1 = std::min<int64_t>(T.jhi, T.klo - 1);
            if (wr1 >= wr0) {
                int cur = -2;
                int64_t c0 = wr0;
                for (int64_t kb = col_block(wr0); kb >= col_block(wr1); --kb) {
                    const int d = dest(I, kb);
                    const int64_t lo = std::max(wr0, n - b - kb * b);
                    if (d != cur) {
                        if (cur != -2) add(src, cur, T.ilo, T.ihi, c0, lo - 1);
                        cur = d, c0 = lo;
                    }
                }
                add(src, cur, T.ilo, T.ihi, c0, wr1);
            }
            // WK: rows [wk0, jhi] x columns K, by row block
            const int64_t wk0 = std::max<int64_t>(T.jlo, T.ihi + 1);
            if (T.jhi >= wk0) {
                int cur = -2;
                int64_t r0 = wk0;
                for (int64_t ia = row_block(wk0); ia <= row_block(T.jhi); ++ia) {
                    const int d = dest(ia, K);
                    const int64_t lo = std::max<int64_t>(wk0, ia ? 1 + (ia - 1) * b : 0);
                    if (d != cur) {
                        if (cur != -2) add(src, cur, r0, lo - 1, T.klo, T.z);
                        cur = d, r0 = lo;
                    }
                }
                add(src, cur, r0, T.jhi, T.klo, T.z);
            }
        }
        // segments of this rank's buffers, pieces grouped by peer
        int64_t so = 0, ro = 0;
        P.sp_off.push_back((int64_t)P.send.size());
        P.rp_off.push_back((int64_t)P.recv.size());
        for (int g = 0; g < world; ++g) {
            P.scnt[r * world + g] = cnt[(size_t)rank * world + g];
            P.rcnt[r * world + g] = cnt[(size_t)g * world + rank];
            P.soff[r * world + g] = so;
            P.roff[r * world + g] = ro;
            for (PieceDesc pc : sp[(size_t)g]) pc.off += so, P.send.push_back(pc);
            for (PieceDesc pc : rp[(size_t)g]) pc.off += ro, P.recv.push_back(pc);
            so += P.scnt[r * world + g];
            ro += P.rcnt[r * world + g];
        }
        P.sp_cnt.push_back((int64_t)P.send.size() - P.sp_off.back());
        P.rp_cnt.push_back((int64_t)P.recv.size() - P.rp_off.back());
        P.send_max = std::max(P.send_max, so);
        P.recv_max = std::max(P.recv_max, ro);
        P.sent += so;
        P.received += ro;
        for (int64_t v : cnt) P.round_any[r] |= v > 0;
    }
}

}  // namespace

extern "C" {

int mp_shard(mp_handle *h, int32_t world, int32_t rank, const void *nccl_id) {
    g_err.clear();
    if (!h || world < 1 || rank < 0 || rank >= world) return fail(MP_ERR_ARG, "bad argument");
    if (h->sh.on) return fail(MP_ERR_ARG, "session is already sharded");
    if (h->kind == MP_SCHEDULE_SERIAL)
        return fail(MP_ERR_UNSUPPORTED, "sharding needs the tiled or diagonal schedule");
    if (h->pass_index != 0 || h->nnz != 0) return fail(MP_ERR_ARG, "shard a session before its first pass");
    CK(cudaSetDevice(h->dev));
    auto &S = h->sh;
    // The communicator first: nothing of the session has changed if NCCL is
    // missing or the rendezvous fails.  (A 1-rank communicator too: it
    // exercises the same set-up.)
    ncclComm_t comm = nullptr;
    if (nccl_id) {
        const NcclApi &N = nccl_api();
        if (!N.commInitRank) return fail(MP_ERR_UNSUPPORTED, "NCCL unavailable: %s", N.why.c_str());
        ncclUniqueId u;
        std::memcpy(&u, nccl_id, sizeof(u));
        NCK(N.commInitRank(&comm, world, u, rank));
    }
    // Any later failure leaves the session as it was: shard buffers freed, the
    // communicator destroyed, the unsharded plan (dataflow launch included) back.
    const bool was_df_allowed = h->df_allowed;
    bool replanned = false;
    auto undo = [&](int rc) {
        const std::string why = g_err;
        cudaGetLastError();
        cudaFree(S.d_my_tiles);
        cudaFree(S.d_send_pc);
        cudaFree(S.d_recv_pc);
        cudaFree(S.sendbuf);
        cudaFree(S.recvbuf);
        cudaFree(S.d_local);
        if (S.h_local) cudaFreeHost(S.h_local);
        if (comm) nccl_api().commDestroy(comm);
        S = mp_handle::Shard();
        h->df_allowed = was_df_allowed;
        if (replanned) replan(h, h->round_cnt);
        g_err = why;
        return rc;
    };
#define TRY_SHARD(call)                                                                      \
    do {                                                                                     \
        const cudaError_t e_ = (call);                                                       \
        if (e_ != cudaSuccess)                                                               \
            return undo(fail(e_ == cudaErrorMemoryAllocation ? MP_ERR_OOM : MP_ERR_CUDA,     \
                             "mp_shard: %s", cudaGetErrorString(e_)));                       \
    } while (0)
    std::vector<int64_t> tz;
    for (const TileDesc &t : h->tiles) tz.push_back(t.z);
    lpt_owner(h->b, world, h->tile_x, tz, h->round_cnt, S.owner);
    // re-plan the launch shapes for the tiles one rank runs per round (the
    // largest share over ranks, so every rank numbers the dual streams alike):
    // fewer tiles per device leave room for larger clusters
    // sharded passes exchange footprints after every round: no dataflow launch
    const bool was_df = h->df_on;
    h->df_allowed = false;
    if (world > 1 || was_df) {
        std::vector<int64_t> share(h->round_cnt.size(), 0);
        for (size_t r = 0; r < h->round_cnt.size(); ++r) {
            std::vector<int64_t> per((size_t)world, 0);
            for (int64_t t = h->round_off[r]; t < h->round_off[r] + h->round_cnt[r]; ++t)
                per[(size_t)S.owner[(size_t)t]]++;
            share[r] = *std::max_element(per.begin(), per.end());
        }
        replanned = true;
        if (int rc = replan(h, share)) return undo(rc);
    }
    std::vector<TileDesc> mine;
    for (size_t r = 0; r < h->round_cnt.size(); ++r) {
        S.my_off.push_back((int64_t)mine.size());
        for (int64_t t = h->round_off[r]; t < h->round_off[r] + h->round_cnt[r]; ++t)
            if (S.owner[(size_t)t] == rank) mine.push_back(h->tiles[(size_t)t]);
        S.my_cnt.push_back((int64_t)mine.size() - S.my_off.back());
    }
    ExchangePlan P;
    plan_exchange(h, S.owner, world, rank, P);
    S.sp_off = P.sp_off, S.sp_cnt = P.sp_cnt, S.rp_off = P.rp_off, S.rp_cnt = P.rp_cnt;
    S.scnt = P.scnt, S.soff = P.soff, S.rcnt = P.rcnt, S.roff = P.roff;
    S.round_any = P.round_any;
    S.sent_per_pass = P.sent, S.recv_per_pass = P.received;
    TRY_SHARD(cudaMalloc(&S.d_my_tiles, std::max<size_t>(mine.size(), 1) * sizeof(TileDesc)));
    if (!mine.empty())
        TRY_SHARD(cudaMemcpy(S.d_my_tiles, mine.data(), mine.size() * sizeof(TileDesc), cudaMemcpyHostToDevice));
    if (world > 1) {
        TRY_SHARD(cudaMalloc(&S.d_send_pc, std::max<size_t>(P.send.size(), 1) * sizeof(PieceDesc)));
        TRY_SHARD(cudaMalloc(&S.d_recv_pc, std::max<size_t>(P.recv.size(), 1) * sizeof(PieceDesc)));
        if (!P.send.empty())
            TRY_SHARD(cudaMemcpy(S.d_send_pc, P.send.data(), P.send.size() * sizeof(PieceDesc), cudaMemcpyHostToDevice));
        if (!P.recv.empty())
            TRY_SHARD(cudaMemcpy(S.d_recv_pc, P.recv.data(), P.recv.size() * sizeof(PieceDesc), cudaMemcpyHostToDevice));
        TRY_SHARD(cudaMalloc(&S.sendbuf, (size_t)std::max<int64_t>(P.send_max, 1) * sizeof(double)));
        TRY_SHARD(cudaMalloc(&S.recvbuf, (size_t)std::max<int64_t>(P.recv_max, 1) * sizeof(double)));
    }
    TRY_SHARD(cudaMalloc(&S.d_local, sizeof(PassCounters)));
    TRY_SHARD(cudaMallocHost(&S.h_local, sizeof(PassCounters)));
#undef TRY_SHARD
    std::memset(S.h_local, 0, sizeof(PassCounters));
    S.world = world;
    S.rank = rank;
    S.local = nccl_id == nullptr;
    S.comm = comm;
    S.on = true;
    return MP_OK;
}

int mp_shard_volume(mp_handle *h, int64_t *sent, int64_t *received) {
    g_err.clear();
    if (!h || !sent || !received) return fail(MP_ERR_ARG, "bad argument");
    *sent = h->sh.on ? h->sh.sent_per_pass : 0;
    *received = h->sh.on ? h->sh.recv_per_pass : 0;
    return MP_OK;
}

int mp_shard_route(int64_t n, int32_t b, int32_t world, int64_t *vol, int64_t *nrounds) {
    g_err.clear();
    if (n < 3 || b < 1 || world < 1 || !nrounds) return fail(MP_ERR_ARG, "bad argument");
    mp_handle h;  // host fields only: the schedule
    h.dev = -1;
    h.n = n;
    h.b = b;
    h.kind = MP_SCHEDULE_TILED;
    std::vector<int64_t> tz;
    enumerate_tiles(n, b, h.tile_x, tz, h.round_cnt);
    *nrounds = (int64_t)h.round_cnt.size();
    if (!vol) return MP_OK;
    h.nib = (n + b - 1) / b + 2;
    h.nkb = (n - 1) / b + 2;
    h.tile_of_blk.assign((size_t)(h.nib * h.nkb), -1);
    int64_t off = 0;
    for (int64_t cnt : h.round_cnt) {
        h.round_off.push_back(off);
        off += cnt;
    }
    for (size_t t = 0; t < tz.size(); ++t) {
        const TileDesc T = make_tile(h.tile_x[t], tz[t], b);
        h.tile_of_blk[(size_t)(((T.ilo + b - 1) / b) * h.nkb + (n - 1 - tz[t]) / b)] = (int32_t)t;
        h.tiles.push_back(T);
    }
    std::vector<int32_t> owner;
    lpt_owner(b, world, h.tile_x, tz, h.round_cnt, owner);
    ExchangePlan P;
    plan_exchange(&h, owner, world, 0, P);
    std::copy(P.pairs.begin(), P.pairs.end(), vol);
    return MP_OK;
}

int mp_group_run_passes(mp_handle *const *hs, int32_t world, int32_t npasses, mp_pass_stats *out) {
    g_err.clear();
    if (!hs || world < 1 || npasses < 0 || (npasses > 0 && !out)) return fail(MP_ERR_ARG, "bad argument");
    std::vector<mp_handle *> v((size_t)world, nullptr);
    for (int32_t g = 0; g < world; ++g) {
        mp_handle *h = hs[g];
        if (!h || !h->sh.on || !h->sh.local || h->sh.world != world)
            return fail(MP_ERR_ARG, "member %d is not a local shard of a %d-way group", g, world);
        if (v[(size_t)h->sh.rank]) return fail(MP_ERR_ARG, "rank %d appears twice", h->sh.rank);
        if (h->dev != hs[0]->dev || h->n != hs[0]->n || h->b != hs[0]->b ||
            h->pass_index != hs[0]->pass_index)
            return fail(MP_ERR_ARG, "group members differ in device, instance size, tile size or pass");
        v[(size_t)h->sh.rank] = h;
    }
    CK(cudaSetDevice(v[0]->dev));
    // one stream for the whole group: the members' kernels run one after the
    // other, none waits on another
    std::vector<cudaStream_t> own;
    for (mp_handle *h : v) {
        own.push_back(h->st);
        h->st = v[0]->st;
    }
    const int rc = run_group(v, npasses, out);
    for (size_t g = 0; g < v.size(); ++g) v[g]->st = own[g];
    return rc;
}

}  // extern "C"

namespace {
__global__ void check_div_kernel(double b, double rb, uint64_t seed, int64_t samples,
                                 unsigned long long *bad) {
    unsigned long long nbad = 0;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < samples;
         t += (int64_t)gridDim.x * blockDim.x) {
        // splitmix64 -> random double across many binades, both signs
        uint64_t z = seed + (uint64_t)t * 0x9E3779B97F4A7C15ull;
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        z ^= z >> 31;
        // |a| in ~[2^-40, 2^40), and every 16th sample across [2^-1000, 2^1000)
        // (the fast path's edges and the IEEE fallback)
        const int ex = (t & 15) == 0 ? (int)((z >> 52) % 2000) - 1000 : (int)((z >> 52) % 80) - 40;
        const double mant = __longlong_as_double((long long)((z & 0xFFFFFFFFFFFFFull) | 0x3FF0000000000000ull));
        double a = ldexp(mant, ex);
        if (z & (1ull << 63)) a = -a;
        if (div_rn(a, b, rb) != __ddiv_rn(a, b)) ++nbad;
    }
    if (nbad) atomicAdd(bad, nbad);
}
}  // namespace

extern "C" {

int mp_check_division(double divisor, int64_t samples, uint64_t seed, int64_t *mismatches) {
    g_err.clear();
    if (!mismatches || !(divisor > 0.0)) return fail(MP_ERR_ARG, "bad argument");
    unsigned long long *d = nullptr;
    CK(cudaMalloc(&d, sizeof(*d)));
    cudaMemset(d, 0, sizeof(*d));
    check_div_kernel<<<148 * 8, 256>>>(divisor, 1.0 / divisor, seed, samples, d);
    unsigned long long hbad = 0;
    cudaError_t e = cudaMemcpy(&hbad, d, sizeof(hbad), cudaMemcpyDeviceToHost);
    cudaFree(d);
    if (e != cudaSuccess) return fail(MP_ERR_CUDA, "check_division: %s", cudaGetErrorString(e));
    *mismatches = (int64_t)hbad;
    return MP_OK;
}

int mp_cc_instance(int64_t n, const int64_t *rowptr, const int32_t *cols, double guard, double cap,
                   double offset, double *d_flat, double *w_flat) {
    g_err.clear();
    if (n < 3) return fail(MP_ERR_ARG, "need at least 3 nodes, got %lld", (long long)n);
    if (!(offset > 0.0)) return fail(MP_ERR_ARG, "sign offset must be positive, got %g", offset);
    if (!rowptr || !d_flat || !w_flat || (rowptr[n] > 0 && !cols)) return fail(MP_ERR_ARG, "bad argument");
    const int64_t nnz = rowptr[n];
    for (int64_t u = 0; u < n; ++u)
        if (rowptr[u + 1] < rowptr[u]) return fail(MP_ERR_ARG, "rowptr must be non-decreasing");
    for (int64_t e = 0; e < nnz; ++e)
        if (cols[e] < 0 || cols[e] >= n) return fail(MP_ERR_ARG, "neighbour index out of range");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
        return fail(MP_ERR_CUDA, "no CUDA device available; there is no CPU fallback");
    const int64_t m = pair_count(n);
    int64_t *drow = nullptr;
    int32_t *dcol = nullptr;
    uint32_t *inter = nullptr;
    double *dd = nullptr, *dw = nullptr;
    cudaStream_t st;
    CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    auto cleanup = [&]() {
        cudaFree(drow);
        cudaFree(dcol);
        cudaFree(inter);
        cudaFree(dd);
        cudaFree(dw);
        cudaStreamDestroy(st);
    };
    cudaError_t e = cudaSuccess;
    if ((e = cudaMalloc(&drow, (size_t)(n + 1) * sizeof(int64_t))) != cudaSuccess ||
        (e = cudaMalloc(&dcol, (size_t)std::max<int64_t>(nnz, 1) * sizeof(int32_t))) != cudaSuccess ||
        (e = cudaMalloc(&inter, (size_t)m * sizeof(uint32_t))) != cudaSuccess ||
        (e = cudaMalloc(&dd, (size_t)m * sizeof(double))) != cudaSuccess ||
        (e = cudaMalloc(&dw, (size_t)m * sizeof(double))) != cudaSuccess) {
        cleanup();
        return fail(MP_ERR_OOM, "cudaMalloc: %s", cudaGetErrorString(e));
    }
    cudaMemcpyAsync(drow, rowptr, (size_t)(n + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, st);
    if (nnz) cudaMemcpyAsync(dcol, cols, (size_t)nnz * sizeof(int32_t), cudaMemcpyHostToDevice, st);
    cudaMemsetAsync(inter, 0, (size_t)m * sizeof(uint32_t), st);
    cc_inter_kernel<<<(unsigned)((n * 32 + 255) / 256), 256, 0, st>>>(drow, dcol, n, inter);
    cc_map_kernel<<<grid_for(m, 256, 148 * 16), 256, 0, st>>>(inter, drow, n, m, guard, cap, offset, dd, dw);
    cudaMemcpyAsync(d_flat, dd, (size_t)m * sizeof(double), cudaMemcpyDeviceToHost, st);
    cudaMemcpyAsync(w_flat, dw, (size_t)m * sizeof(double), cudaMemcpyDeviceToHost, st);
    e = cudaStreamSynchronize(st);
    if (e == cudaSuccess) e = cudaGetLastError();
    cleanup();
    if (e != cudaSuccess) return fail(MP_ERR_CUDA, "cc_instance: %s", cudaGetErrorString(e));
    return MP_OK;
}

int mp_max_violation(int64_t n, const double *xv, const double *fv, const double *d_flat,
                     double *out) {
    g_err.clear();
    if (n < 3 || !xv || !fv || !d_flat || !out) return fail(MP_ERR_ARG, "bad argument");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
        return fail(MP_ERR_CUDA, "no CUDA device available; there is no CPU fallback");
    const int64_t m = pair_count(n), ld = (n + 31) / 32 * 32;
    double *dx = nullptr, *px = nullptr, *pf = nullptr, *pd = nullptr;
    unsigned long long *acc = nullptr;
    cudaStream_t st;
    CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    auto cleanup = [&]() {
        cudaFree(dx);
        cudaFree(px);
        cudaFree(pf);
        cudaFree(pd);
        cudaFree(acc);
        cudaStreamDestroy(st);
    };
    cudaError_t e = cudaSuccess;
    if ((e = cudaMalloc(&dx, (size_t)n * ld * sizeof(double))) != cudaSuccess ||
        (e = cudaMalloc(&px, m * sizeof(double))) != cudaSuccess ||
        (e = cudaMalloc(&pf, m * sizeof(double))) != cudaSuccess ||
        (e = cudaMalloc(&pd, m * sizeof(double))) != cudaSuccess ||
        (e = cudaMalloc(&acc, sizeof(unsigned long long))) != cudaSuccess) {
        cleanup();
        return fail(MP_ERR_OOM, "cudaMalloc: %s", cudaGetErrorString(e));
    }
    cudaMemcpyAsync(px, xv, m * sizeof(double), cudaMemcpyHostToDevice, st);
    cudaMemcpyAsync(pf, fv, m * sizeof(double), cudaMemcpyHostToDevice, st);
    cudaMemcpyAsync(pd, d_flat, m * sizeof(double), cudaMemcpyHostToDevice, st);
    cudaMemsetAsync(acc, 0, sizeof(unsigned long long), st);
    const int g = grid_for(m, 256, 148 * 16);
    expand_kernel<<<g, 256, 0, st>>>(px, dx, ld, n, m);
    scan_metric_kernel<<<(unsigned)(n - 2), 256, 0, st>>>(dx, ld, n, acc);
    scan_pair_kernel<<<g, 256, 0, st>>>(dx, ld, pf, pd, n, m, acc);
    unsigned long long bits = 0;
    cudaMemcpyAsync(&bits, acc, sizeof(bits), cudaMemcpyDeviceToHost, st);
    e = cudaStreamSynchronize(st);
    cleanup();
    if (e != cudaSuccess) return fail(MP_ERR_CUDA, "max_violation: %s", cudaGetErrorString(e));
    double v;
    std::memcpy(&v, &bits, sizeof(v));
    *out = v;
    return MP_OK;
}

int mp_dykstra_steps(int64_t nrows, const int32_t *nent, const int64_t *pos, const double *coef,
                     const double *reg, const double *rhs, const double *y_old, double eps,
                     int64_t nv, double *v, double *theta, int32_t *changed) {
    g_err.clear();
    if (nrows < 0 || nv < 0 || (nrows > 0 && (!nent || !pos || !coef || !reg || !rhs || !y_old ||
                                              !v || !theta || !changed)))
        return fail(MP_ERR_ARG, "bad argument");
    if (!(eps > 0.0)) return fail(MP_ERR_ARG, "epsilon must be positive, got %g", eps);
    if (nrows == 0) return MP_OK;
    std::vector<StepRow> rows((size_t)nrows);
    for (int64_t r = 0; r < nrows; ++r) {
        if (nent[r] != 2 && nent[r] != 3) return fail(MP_ERR_ARG, "row %lld: %d entries", (long long)r, nent[r]);
        if (!(y_old[r] >= 0.0))
            return fail(MP_ERR_ARG, "dual values are nonnegative, got %g", y_old[r]);
        StepRow &R = rows[(size_t)r];
        R.nent = nent[r];
        R.pad = 0;
        for (int e = 0; e < 3; ++e) {
            const bool on = e < nent[r];
            R.pos[e] = on ? pos[3 * r + e] : 0;
            R.coef[e] = on ? coef[3 * r + e] : 0.0;
            R.reg[e] = on ? reg[3 * r + e] : 1.0;
            if (on && (R.pos[e] < 0 || R.pos[e] >= nv))
                return fail(MP_ERR_ARG, "row %lld: position out of range", (long long)r);
        }
        R.rhs = rhs[r];
        R.y = y_old[r];
    }
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
        return fail(MP_ERR_CUDA, "no CUDA device available; there is no CPU fallback");
    StepRow *drows = nullptr;
    double *dv = nullptr, *dth = nullptr;
    int32_t *dch = nullptr;
    cudaStream_t st;
    CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    auto cleanup = [&]() {
        cudaFree(drows);
        cudaFree(dv);
        cudaFree(dth);
        cudaFree(dch);
        cudaStreamDestroy(st);
    };
    cudaError_t e = cudaSuccess;
    if ((e = cudaMalloc(&drows, rows.size() * sizeof(StepRow))) != cudaSuccess ||
        (e = cudaMalloc(&dv, (size_t)std::max<int64_t>(nv, 1) * sizeof(double))) != cudaSuccess ||
        (e = cudaMalloc(&dth, (size_t)nrows * sizeof(double))) != cudaSuccess ||
        (e = cudaMalloc(&dch, (size_t)nrows * sizeof(int32_t))) != cudaSuccess) {
        cleanup();
        return fail(MP_ERR_OOM, "cudaMalloc: %s", cudaGetErrorString(e));
    }
    cudaMemcpyAsync(drows, rows.data(), rows.size() * sizeof(StepRow), cudaMemcpyHostToDevice, st);
    cudaMemcpyAsync(dv, v, (size_t)nv * sizeof(double), cudaMemcpyHostToDevice, st);
    single_steps_kernel<<<1, 32, 0, st>>>(drows, nrows, eps, dv, dth, dch);
    cudaMemcpyAsync(v, dv, (size_t)nv * sizeof(double), cudaMemcpyDeviceToHost, st);
    cudaMemcpyAsync(theta, dth, (size_t)nrows * sizeof(double), cudaMemcpyDeviceToHost, st);
    cudaMemcpyAsync(changed, dch, (size_t)nrows * sizeof(int32_t), cudaMemcpyDeviceToHost, st);
    e = cudaStreamSynchronize(st);
    if (e == cudaSuccess) e = cudaGetLastError();
    cleanup();
    if (e != cudaSuccess) return fail(MP_ERR_CUDA, "dykstra_steps: %s", cudaGetErrorString(e));
    return MP_OK;
}

int mp_accumulate_aty(int64_t n, int64_t nnz, const int64_t *keys, const double *vals,
                      const double *pair_duals, const double *c, double *g) {
    g_err.clear();
    if (n < 3 || nnz < 0 || (nnz > 0 && (!keys || !vals)) || !pair_duals || !c || !g)
        return fail(MP_ERR_ARG, "bad argument");
    const int64_t m = pair_count(n);
    if (2 * m > (int64_t)UINT32_MAX || 3 * nnz > (int64_t)INT32_MAX)
        return fail(MP_ERR_ARG, "accumulate_aty: sizes beyond 32-bit record indices");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
        return fail(MP_ERR_CUDA, "no CUDA device available; there is no CPU fallback");
    const int nrec = (int)(3 * nnz);
    int end_bit = 1;
    while (end_bit < 32 && ((int64_t)1 << end_bit) < m) ++end_bit;
    double *dg = nullptr, *dc = nullptr, *dpd = nullptr, *dv = nullptr;
    int64_t *dk = nullptr;
    uint32_t *t0 = nullptr, *t1 = nullptr, *r0 = nullptr, *r1 = nullptr;
    int *bad = nullptr;
    void *tmp = nullptr;
    size_t tmp_bytes = 0;
    cudaStream_t st;
    CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    auto cleanup = [&]() {
        for (void *q : {(void *)dg, (void *)dc, (void *)dpd, (void *)dv, (void *)dk, (void *)t0,
                        (void *)t1, (void *)r0, (void *)r1, (void *)bad, tmp})
            cudaFree(q);
        cudaStreamDestroy(st);
    };
    cudaError_t e = cudaSuccess;
    const size_t nr = (size_t)std::max(nrec, 1);
    if (nrec > 0)
        cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, t0, t1, r0, r1, nrec, 0, end_bit, st);
    if ((e = cudaMalloc(&dg, 2 * m * sizeof(double))) != cudaSuccess ||
        (e = cudaMalloc(&dc, 2 * m * sizeof(double))) != cudaSuccess ||
        (e = cudaMalloc(&dpd, 2 * m * sizeof(double))) != cudaSuccess ||
        (e = cudaMalloc(&dv, std::max<int64_t>(nnz, 1) * sizeof(double))) != cudaSuccess ||
        (e = cudaMalloc(&dk, std::max<int64_t>(nnz, 1) * sizeof(int64_t))) != cudaSuccess ||
        (e = cudaMalloc(&t0, nr * 4)) != cudaSuccess || (e = cudaMalloc(&t1, nr * 4)) != cudaSuccess ||
        (e = cudaMalloc(&r0, nr * 4)) != cudaSuccess || (e = cudaMalloc(&r1, nr * 4)) != cudaSuccess ||
        (e = cudaMalloc(&bad, sizeof(int))) != cudaSuccess ||
        (e = cudaMalloc(&tmp, std::max<size_t>(tmp_bytes, 16))) != cudaSuccess) {
        cleanup();
        return fail(MP_ERR_OOM, "cudaMalloc: %s", cudaGetErrorString(e));
    }
    cudaMemcpyAsync(dc, c, 2 * m * sizeof(double), cudaMemcpyHostToDevice, st);
    cudaMemcpyAsync(dg, dc, m * sizeof(double), cudaMemcpyDeviceToDevice, st);
    cudaMemcpyAsync(dpd, pair_duals, 2 * m * sizeof(double), cudaMemcpyHostToDevice, st);
    cudaMemsetAsync(bad, 0, sizeof(int), st);
    if (nnz > 0) {
        cudaMemcpyAsync(dk, keys, nnz * sizeof(int64_t), cudaMemcpyHostToDevice, st);
        cudaMemcpyAsync(dv, vals, nnz * sizeof(double), cudaMemcpyHostToDevice, st);
        aty_records_kernel<<<grid_for(nnz, 256, 148 * 16), 256, 0, st>>>(dk, nnz, n, t0, r0, bad);
        cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, t0, t1, r0, r1, nrec, 0, end_bit, st);
        aty_segments_kernel<<<grid_for(nrec, 256, 148 * 16), 256, 0, st>>>(t1, r1, nrec, dv, dg);
    }
    aty_pairs_kernel<<<grid_for(m, 256, 148 * 16), 256, 0, st>>>(dpd, dc, dg, m);
    int hbad = 0;
    cudaMemcpyAsync(g, dg, 2 * m * sizeof(double), cudaMemcpyDeviceToHost, st);
    cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, st);
    e = cudaStreamSynchronize(st);
    if (e == cudaSuccess) e = cudaGetLastError();
    cleanup();
    if (e != cudaSuccess) return fail(MP_ERR_CUDA, "accumulate_aty: %s", cudaGetErrorString(e));
    if (hbad) return fail(MP_ERR_ARG, "invalid metric key");
    return MP_OK;
}

}  // extern "C"
