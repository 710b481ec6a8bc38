// pool.cpp -- the C ABI of include/lora_delta.h: paged HBM adapter pool, cold-start
// loader on a side stream, host planner, and the launches of the sm_100a kernels.
//
// Paper anchors: adapters live in host memory and are fetched to the GPU on demand
// (§2.3 C1 P:353-392, §3); the GPU LoRA is batched per layer and
// added to the base output (§4.1); invocation is sync-free, relying on CUDA
// stream order (§4.2).  The paged store follows "optimized GPU memory
// management" borrowed from S-LoRA/LightLLM: one page = one rank
// component (a_j ∈ R^{H_in}, b_j ∈ R^{H_out}) -- DESIGN.md reading R9.
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/lora_delta.h"
#include "kernel_config.h"
#include "plan.h"


using namespace lora;

static thread_local std::string g_err;

static lora_status fail(lora_status s, const std::string& msg) {
    g_err = msg;
    return s;
}

struct lora_pool {
    int H_in = 0, H_out = 0, max_adapters = 0, n_pages = 0, esz = 2, device = 0, num_sms = 148;
    lora_dtype dtype = LORA_BF16;
    unsigned flags = 0;
    bool host_only = false;
    char* dA = nullptr;                  // [n_pages + 1][H_in]  (row n_pages: all-zero page)
    char* dB = nullptr;                  // [n_pages + 1][H_out]
    bool tc_prefill = false;             // tensor-core prefill path available for this pool
    alignas(64) unsigned char tm_a[128]; // TMA maps of the page arrays (gather4 boxes {64, 1})
    alignas(64) unsigned char tm_b[128];
    void* box_maps = nullptr;            // device: 2 x kBoxKinds 2D box tensor maps of the page arrays (TMA boxes)
    std::vector<uint8_t> page_used;
    int free_pages = 0;
    AdapterTable table;
    // cold-start loads round-robin over kSideStreams (8) side streams, so consecutive small loads (PCIe
    // latency-bound one at a time) overlap; ordering against page reuse is by events (unload)
#ifndef LORA_SIDE_STREAMS
#define LORA_SIDE_STREAMS 8   // c4 step: 1 stream 0.513, 4 streams 0.464, 8 streams 0.452 ms
#endif
    static constexpr int kSideStreams = LORA_SIDE_STREAMS;
    cudaStream_t sides[kSideStreams] = {};
    int next_side = 0;
    cudaStream_t side = nullptr;          // == sides[0]
    cudaEvent_t unload_fence = nullptr;
    bool fence_pending = false;
    std::vector<cudaStream_t> apply_streams;   // streams applied on since the last unload
    float* vbuf = nullptr;
    float* pf_scratch = nullptr;         // prefill split-K partials (grown on demand)
    size_t pf_scratch_cap = 0;
    uint16_t* fb_vtiles = nullptr;       // lora_apply_fused_base: V tiles (bf16, grown on demand)
    size_t fb_vtiles_cap = 0;
    int* fb_vsync = nullptr;             // lora_apply_fused_base: launch epochs + per-V-tile flags (zeroed once)
    size_t fb_vsync_cap = 0;
    size_t vbuf_cap = 0;                 // floats
    int32_t* meta_dev = nullptr;
    size_t meta_cap = 0;                 // words
    bool load_kernel = false;            // LORA_OPT_LOAD_KERNEL: cold-start copies by a zero-copy gather kernel
    bool pad_max_rank = false;           // LORA_OPT_PAD_MAX_RANK: BGMV-style padded decode work (comparison)
    Plan plan;
    Plan fused;                          // merged kernel work of the last lora_apply_multi led by this pool
    int L_tc = 64;
    int64_t launches = 0;
    bool split_ready = false;             // a lora_apply_shrink awaits its lora_apply_expand
    unsigned long long* trace = nullptr;   // lora_debug_set_trace
    bool capturing = false;               // the current apply's stream is being captured into a graph
    std::vector<void*> retired;           // outgrown scratch buffers: a captured graph may still use them
    int32_t* gc_cnt = nullptr;            // TP shrink: per-gc arrival counters (zero between applies)
    size_t gc_cnt_cap = 0;
    float* vred = nullptr;                // TP: the compact k-reduced v all-reduced by lora_apply_tp
    size_t vred_cap = 0;
    lora_tp_comm* tp = nullptr;           // lora_tp_init: the TP group's communicator (not owned)
    // plan cache (plan_cached): `plan` is rebuilt only when the batch, the adapter table or a planner
    // setting changed -- a decode batch repeats from step to step, and the library is invoked for
    // every projection of every layer (per-invocation overhead matters)
    uint64_t table_version = 1;           // bumped by every change the planner reads (adapters, options)
    struct PlanKey {
        uint64_t version = 0;             // 0: invalid
        int tc = -1, pad = -1, budget = -1, L_tc = -1;
        std::vector<int32_t> ip, ids;
    } pkey;
    uint64_t plan_gen = 1;                // bumped whenever `plan` is rebuilt
    uint64_t ready_gen = 0;               // == plan_gen: every adapter of `plan` is known loaded
    struct FusedKey {                     // the pools and plan generations `fused` was merged from
        int n = 0;
        const lora_pool* pools[kMaxJobs] = {};
        uint64_t gens[kMaxJobs] = {};
    } fkey;
};

namespace {
// p->plan for (seg_indptr, adapter_ids) under the given planner settings; rebuilt only on a change
lora_status plan_cached(lora_pool* p, const int32_t* ip, const int32_t* ids, int S, bool tc, int pad, int budget,
                        std::string& err) {
    lora_pool::PlanKey& k = p->pkey;
    if (k.version == p->table_version && k.tc == (int)tc && k.pad == pad && k.budget == budget && k.L_tc == p->L_tc &&
        (int)k.ids.size() == S && std::equal(ids, ids + S, k.ids.begin()) && std::equal(ip, ip + S + 1, k.ip.begin()))
        return LORA_OK;
    k.version = 0;
    ++p->plan_gen;
    lora_status s = build_plan(p->plan, ip, ids, S, p->H_in, p->H_out, p->esz, p->L_tc, tc, p->table, err, pad,
                               p->num_sms, budget);
    if (s != LORA_OK) return s;
    k.version = p->table_version;
    k.tc = (int)tc; k.pad = pad; k.budget = budget; k.L_tc = p->L_tc;
    k.ip.assign(ip, ip + S + 1);
    k.ids.assign(ids, ids + S);
    return LORA_OK;
}
// p->plan was (re)built outside plan_cached
void plan_uncached(lora_pool* p) {
    p->pkey.version = 0;
    ++p->plan_gen;
}
}  // namespace

// ---- NCCL, resolved at run time (dlopen): the library loads without NCCL; only the TP calls need it.
// The few types and constants used are NCCL's stable ABI (nccl.h 2.x: ncclUniqueId is 128 bytes,
// ncclSuccess = 0, ncclSum = 0, ncclFloat32 = 7).
namespace {
typedef struct { char internal[LORA_TP_UNIQUE_ID_BYTES]; } nccl_uid;
typedef void* nccl_comm;
struct NcclApi {
    int (*get_unique_id)(nccl_uid*) = nullptr;
    int (*comm_init_rank)(nccl_comm*, int, nccl_uid, int) = nullptr;
    int (*all_reduce)(const void*, void*, size_t, int, int, nccl_comm, cudaStream_t) = nullptr;
    int (*comm_destroy)(nccl_comm) = nullptr;
    const char* (*error_string)(int) = nullptr;
};
const NcclApi* nccl(std::string& err) {
    static NcclApi api;
    static bool tried = false, ok = false;
    if (!tried) {
        tried = true;
        // the process's NCCL (torch loads libnccl.so.2), else the one beside the CUDA runtime
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (h) {
            api.get_unique_id = (int (*)(nccl_uid*))dlsym(h, "ncclGetUniqueId");
            api.comm_init_rank = (int (*)(nccl_comm*, int, nccl_uid, int))dlsym(h, "ncclCommInitRank");
            api.all_reduce = (int (*)(const void*, void*, size_t, int, int, nccl_comm, cudaStream_t))dlsym(h, "ncclAllReduce");
            api.comm_destroy = (int (*)(nccl_comm))dlsym(h, "ncclCommDestroy");
            api.error_string = (const char* (*)(int))dlsym(h, "ncclGetErrorString");
            ok = api.get_unique_id && api.comm_init_rank && api.all_reduce && api.comm_destroy && api.error_string;
        }
    }
    if (!ok) err = std::string("NCCL is not available (dlopen libnccl.so.2: ") + (dlerror() ? dlerror() : "symbols missing") + ")";
    return ok ? &api : nullptr;
}
constexpr int kNcclSum = 0, kNcclFloat32 = 7;
}  // namespace

struct lora_tp_comm {
    nccl_comm comm = nullptr;
    int rank = 0, size = 1, device = 0;
};

namespace {

struct DeviceGuard {
    int prev = -1;
    bool changed = false;
    explicit DeviceGuard(int dev) {
        if (cudaGetDevice(&prev) == cudaSuccess && prev != dev) {
            cudaSetDevice(dev);
            changed = true;
        }
    }
    ~DeviceGuard() {
        if (changed) cudaSetDevice(prev);
    }
};

lora_status cuda_fail(cudaError_t e, const char* what) {
    return fail(LORA_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

#define CUDA_TRY(call, what)                      \
    do {                                          \
        cudaError_t _e = (call);                  \
        if (_e != cudaSuccess) return cuda_fail(_e, what); \
    } while (0)

bool is_pinned(const void* p, const void** dev_ptr = nullptr) {
    cudaPointerAttributes attr;
    if (cudaPointerGetAttributes(&attr, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    if (dev_ptr) *dev_ptr = attr.devicePointer;   // UVA-mapped address for zero-copy reads (or null)
    return attr.type == cudaMemoryTypeHost;
}

// grow a device buffer (rare; synchronises the device so no in-flight kernel uses the old one)
template <typename T>
lora_status grow(lora_pool* p, T*& buf, size_t& cap, size_t need, bool zero, const char* what) {
    if (need <= cap) return LORA_OK;
    // no allocation, synchronisation or free inside a capture: that would invalidate the caller's graph
    if (p->capturing)
        return fail(LORA_ERR_UNSUPPORTED, std::string(what) +
                                              " scratch must grow inside a CUDA graph capture: run this batch shape "
                                              "once outside the capture, or pre-size it with LORA_OPT_RESERVE_TOKENS");
    size_t n = std::max(need, cap * 2);
    T* nb = nullptr;
    CUDA_TRY(cudaMalloc((void**)&nb, n * sizeof(T)), what);
    if (zero) {
        CUDA_TRY(cudaMemset(nb, 0, n * sizeof(T)), what);
        CUDA_TRY(cudaDeviceSynchronize(), what);
    }
    // the old buffer is not freed: in-flight kernels and graphs captured earlier keep its address
    // (freed with the pool; geometric growth bounds the total at twice the final size)
    if (buf) p->retired.push_back(buf);
    buf = nb;
    cap = n;
    return LORA_OK;
}

// order `st` after an adapter's cold-start load.  While `st` is being captured no event may be
// queried (cudaEventQuery invalidates a capture), so the wait becomes an external event-wait node
// (a no-op at replay once the load has completed).
lora_status wait_loaded(AdapterRec& a, cudaStream_t st, bool capturing, const char* what) {
    if (a.ready_known) return LORA_OK;
    if (capturing) {
        CUDA_TRY(cudaStreamWaitEvent(st, (cudaEvent_t)a.ready, cudaEventWaitExternal), what);
        return LORA_OK;
    }
    cudaError_t e = cudaEventQuery((cudaEvent_t)a.ready);
    if (e == cudaSuccess) {
        a.ready_known = true;
        return LORA_OK;
    }
    if (e != cudaErrorNotReady) return cuda_fail(e, what);
    cudaGetLastError();
    CUDA_TRY(cudaStreamWaitEvent(st, (cudaEvent_t)a.ready, 0), what);
    return LORA_OK;
}

}  // namespace

extern "C" {

const char* lora_last_error(void) { return g_err.c_str(); }

int lora_abi_version(void) { return LORA_ABI_VERSION; }

lora_status lora_pool_create_ex(int hidden_in, int hidden_out, int max_adapters, lora_dtype dtype,
                                int max_total_rank, unsigned flags, lora_pool** out) {
    if (!out) return fail(LORA_ERR_ARG, "out is NULL");
    *out = nullptr;
    if (dtype != LORA_F32 && dtype != LORA_BF16) return fail(LORA_ERR_ARG, "dtype must be LORA_F32 or LORA_BF16");
    if (hidden_in <= 0 || hidden_out <= 0) return fail(LORA_ERR_SHAPE, "hidden_in/hidden_out must be > 0");
    if (max_adapters <= 0) return fail(LORA_ERR_SHAPE, "max_adapters must be > 0");
    if (max_total_rank < 0) return fail(LORA_ERR_SHAPE, "max_total_rank must be >= 0");
    const int esz = dtype == LORA_BF16 ? 2 : 4;
    const int vec = 16 / esz;
    if (hidden_in % vec || hidden_out % vec)
        return fail(LORA_ERR_ALIGN, "hidden_in and hidden_out must be multiples of " + std::to_string(vec));
    lora_pool* p = new lora_pool();
    p->H_in = hidden_in;
    p->H_out = hidden_out;
    p->max_adapters = max_adapters;
    p->n_pages = max_total_rank > 0 ? max_total_rank : 64 * max_adapters;
    p->dtype = dtype;
    p->esz = esz;
    p->flags = flags;
    p->host_only = (flags & LORA_POOL_HOST_ONLY) != 0;
    p->page_used.assign(p->n_pages, 0);
    p->free_pages = p->n_pages;
    if (!p->host_only) {
        cudaError_t e = cudaGetDevice(&p->device);
        if (e == cudaSuccess) e = cudaDeviceGetAttribute(&p->num_sms, cudaDevAttrMultiProcessorCount, p->device);
        if (e == cudaSuccess) e = cudaMalloc((void**)&p->dA, (size_t)(p->n_pages + 1) * hidden_in * esz);
        if (e == cudaSuccess) e = cudaMalloc((void**)&p->dB, (size_t)(p->n_pages + 1) * hidden_out * esz);
        if (e == cudaSuccess) e = cudaMemset(p->dA + (size_t)p->n_pages * hidden_in * esz, 0, (size_t)hidden_in * esz);
        if (e == cudaSuccess) e = cudaMemset(p->dB + (size_t)p->n_pages * hidden_out * esz, 0, (size_t)hidden_out * esz);
        if (e == cudaSuccess && prefill_supported(hidden_in, hidden_out, esz)) {
            p->tc_prefill = make_tmap_bf16(p->tm_a, p->dA, p->n_pages + 1, hidden_in, 1) == 0 &&
                            make_tmap_bf16(p->tm_b, p->dB, p->n_pages + 1, hidden_out, 1) == 0;
        }
        // page contents start zeroed (rows a TMA box loads past an adapter are then finite)
        if (e == cudaSuccess) e = cudaMemset(p->dA, 0, (size_t)(p->n_pages + 1) * hidden_in * esz);
        if (e == cudaSuccess) e = cudaMemset(p->dB, 0, (size_t)(p->n_pages + 1) * hidden_out * esz);
        if (e == cudaSuccess && p->tc_prefill) {
            alignas(64) unsigned char maps[2 * kBoxKinds * 128];
            if (make_box_tmaps(maps, p->dA, p->dB, p->n_pages + 1, hidden_in, hidden_out) == 0) {
                e = cudaMalloc(&p->box_maps, sizeof(maps));
                if (e == cudaSuccess) e = cudaMemcpy(p->box_maps, maps, sizeof(maps), cudaMemcpyHostToDevice);
            }
        }
        for (int i = 0; i < lora_pool::kSideStreams && e == cudaSuccess; ++i)
            e = cudaStreamCreateWithFlags(&p->sides[i], cudaStreamNonBlocking);
        p->side = p->sides[0];
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&p->unload_fence, cudaEventDisableTiming);
        if (e != cudaSuccess) {
            lora_pool_destroy(p);
            return cuda_fail(e, "lora_pool_create");
        }
    }
    *out = p;
    return LORA_OK;
}

lora_status lora_pool_create(int hidden_in, int hidden_out, int max_adapters, lora_dtype dtype,
                             int max_total_rank, lora_pool** out) {
    return lora_pool_create_ex(hidden_in, hidden_out, max_adapters, dtype, max_total_rank, 0u, out);
}

lora_status lora_pool_destroy(lora_pool* p) {
    if (!p) return LORA_OK;
    if (!p->host_only) {
        DeviceGuard g(p->device);
        for (cudaStream_t s : p->sides)
            if (s) cudaStreamSynchronize(s);
        for (cudaStream_t s : p->apply_streams) cudaStreamSynchronize(s);
        cudaDeviceSynchronize();
        for (auto& kv : p->table)
            if (kv.second.ready) cudaEventDestroy((cudaEvent_t)kv.second.ready);
        if (p->dA) cudaFree(p->dA);
        if (p->box_maps) cudaFree(p->box_maps);
        if (p->dB) cudaFree(p->dB);
        if (p->vbuf) cudaFree(p->vbuf);
        if (p->vred) cudaFree(p->vred);
        if (p->gc_cnt) cudaFree(p->gc_cnt);
        if (p->pf_scratch) cudaFree(p->pf_scratch);
        if (p->fb_vtiles) cudaFree(p->fb_vtiles);
        if (p->fb_vsync) cudaFree(p->fb_vsync);
        if (p->meta_dev) cudaFree(p->meta_dev);
        for (void* b : p->retired) cudaFree(b);
        if (p->unload_fence) cudaEventDestroy(p->unload_fence);
        for (cudaStream_t s : p->sides)
            if (s) cudaStreamDestroy(s);
    }
    delete p;
    return LORA_OK;
}

// a_pitch / b_pitch: bytes between consecutive rank rows of the host buffers (0 = the pool's row
// bytes, i.e. a contiguous [rank][hidden] buffer; larger for a TP shard of the full adapter)
static lora_status load_impl(lora_pool* p, int32_t id, int rank, const void* A_host, size_t a_pitch, const void* B_host,
                             size_t b_pitch, float scale) {
    if (!p) return fail(LORA_ERR_ARG, "pool is NULL");
    if (id < 0) return fail(LORA_ERR_ARG, "id must be >= 0");
    const int rmax = std::min(LORA_MAX_RANK, std::min(p->H_in, p->H_out));
    if (rank < 1 || rank > rmax)
        return fail(LORA_ERR_SHAPE, "rank " + std::to_string(rank) + " outside [1, " + std::to_string(rmax) + "]");
    if (p->table.count(id)) return fail(LORA_ERR_EXISTS, "adapter " + std::to_string(id) + " already loaded");
    if ((int)p->table.size() >= p->max_adapters) return fail(LORA_ERR_POOL_FULL, "adapter slots exhausted");
    if (p->free_pages < rank)
        return fail(LORA_ERR_POOL_FULL, "page budget exhausted: need " + std::to_string(rank) + ", free " +
                                            std::to_string(p->free_pages));
    const void* devA = nullptr;
    const void* devB = nullptr;
    if (!p->host_only) {
        if (!A_host || !B_host) return fail(LORA_ERR_ARG, "A_host/B_host is NULL");
        if (!is_pinned(A_host, &devA)) return fail(LORA_ERR_NOT_PINNED, "A_host is not pinned host memory");
        if (!is_pinned(B_host, &devB)) return fail(LORA_ERR_NOT_PINNED, "B_host is not pinned host memory");
    }
    // lowest free pages, ascending (reading R9)
    AdapterRec rec;
    rec.id = id;
    rec.rank = rank;
    rec.scale = scale;
    rec.pages.reserve(rank);
    for (int pg = 0; pg < p->n_pages && (int)rec.pages.size() < rank; ++pg)
        if (!p->page_used[pg]) rec.pages.push_back(pg);
    if (!p->host_only) {
        DeviceGuard g(p->device);
        cudaEvent_t ev = nullptr;
        CUDA_TRY(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming), "lora_load_adapter: event");
        cudaStream_t ss = p->sides[p->next_side];
        p->next_side = (p->next_side + 1) % lora_pool::kSideStreams;
        if (p->fence_pending) {
            cudaError_t e = cudaStreamWaitEvent(ss, p->unload_fence, 0);
            if (e != cudaSuccess) { cudaEventDestroy(ev); return cuda_fail(e, "lora_load_adapter: fence"); }
            p->fence_pending = false;
        }
        const size_t ra = (size_t)p->H_in * p->esz, rb = (size_t)p->H_out * p->esz;
        const bool strided = (a_pitch && a_pitch != ra) || (b_pitch && b_pitch != rb);
        if (!a_pitch) a_pitch = ra;
        if (!b_pitch) b_pitch = rb;
        if (strided) {
            // a TP shard: one 2D copy per run of consecutive pages, straight from the full pinned
            // adapter (no host-side slice or re-pin on the cold-start path)
            for (int j = 0; j < rank;) {
                int k = j + 1;
                while (k < rank && rec.pages[k] == rec.pages[k - 1] + 1) ++k;
                cudaError_t e = cudaMemcpy2DAsync(p->dA + (size_t)rec.pages[j] * ra, ra, (const char*)A_host + j * a_pitch,
                                                  a_pitch, ra, (size_t)(k - j), cudaMemcpyHostToDevice, ss);
                if (e == cudaSuccess)
                    e = cudaMemcpy2DAsync(p->dB + (size_t)rec.pages[j] * rb, rb, (const char*)B_host + j * b_pitch, b_pitch,
                                          rb, (size_t)(k - j), cudaMemcpyHostToDevice, ss);
                if (e != cudaSuccess) { cudaEventDestroy(ev); return cuda_fail(e, "lora_load_adapter_shard: copy"); }
                j = k;
            }
        } else if (p->load_kernel && devA && devB && ((uintptr_t)devA % 16) == 0 && ((uintptr_t)devB % 16) == 0) {
            // zero-copy gather kernel (LORA_OPT_LOAD_KERNEL)
            cudaError_t e = (cudaError_t)launch_load(p->dA, p->dB, devA, devB, (int64_t)ra, (int64_t)rb, rank,
                                                     rec.pages.data(), p->num_sms, ss);
            if (e != cudaSuccess) { cudaEventDestroy(ev); return cuda_fail(e, "lora_load_adapter: load kernel"); }
        } else
        // one copy per run of consecutive pages
        for (int j = 0; j < rank;) {
            int k = j + 1;
            while (k < rank && rec.pages[k] == rec.pages[k - 1] + 1) ++k;
            const size_t n = (size_t)(k - j);
            cudaError_t e = cudaMemcpyAsync(p->dA + (size_t)rec.pages[j] * ra, (const char*)A_host + j * ra, n * ra,
                                            cudaMemcpyHostToDevice, ss);
            if (e == cudaSuccess)
                e = cudaMemcpyAsync(p->dB + (size_t)rec.pages[j] * rb, (const char*)B_host + j * rb, n * rb,
                                    cudaMemcpyHostToDevice, ss);
            if (e != cudaSuccess) { cudaEventDestroy(ev); return cuda_fail(e, "lora_load_adapter: copy"); }
            j = k;
        }
        cudaError_t e = cudaEventRecord(ev, ss);
        if (e != cudaSuccess) { cudaEventDestroy(ev); return cuda_fail(e, "lora_load_adapter: record"); }
        rec.ready = ev;
    } else {
        rec.ready_known = true;
    }
    for (int pg : rec.pages) p->page_used[pg] = 1;
    p->free_pages -= rank;
    p->table.emplace(id, std::move(rec));
    ++p->table_version;
    return LORA_OK;
}

lora_status lora_load_adapter(lora_pool* p, int32_t id, int rank, const void* A_host, const void* B_host,
                              float scale) {
    return load_impl(p, id, rank, A_host, 0, B_host, 0, scale);
}

lora_status lora_load_adapter_shard(lora_pool* p, int32_t id, int rank, const void* A_host, int64_t a_ld, int64_t a_col0,
                                    const void* B_host, int64_t b_ld, int64_t b_col0, float scale) {
    if (!p) return fail(LORA_ERR_ARG, "pool is NULL");
    if (a_col0 < 0 || b_col0 < 0 || a_ld < a_col0 + p->H_in || b_ld < b_col0 + p->H_out)
        return fail(LORA_ERR_SHAPE, "shard columns outside the full adapter (a_ld/b_ld too small)");
    if (((a_ld | a_col0) * p->esz) % 16 || ((b_ld | b_col0) * p->esz) % 16)
        return fail(LORA_ERR_ALIGN, "shard row pitch and first column must be 16-B aligned");
    const char* A = A_host ? (const char*)A_host + a_col0 * p->esz : nullptr;
    const char* B = B_host ? (const char*)B_host + b_col0 * p->esz : nullptr;
    return load_impl(p, id, rank, A, (size_t)a_ld * p->esz, B, (size_t)b_ld * p->esz, scale);
}

lora_status lora_unload_adapter(lora_pool* p, int32_t id) {
    if (!p) return fail(LORA_ERR_ARG, "pool is NULL");
    auto it = p->table.find(id);
    if (it == p->table.end()) return fail(LORA_ERR_UNKNOWN_ADAPTER, "adapter " + std::to_string(id) + " is not loaded");
    if (!p->host_only) {
        DeviceGuard g(p->device);
        // physical reuse of these pages must follow every apply already enqueued (events)
        for (cudaStream_t s : p->apply_streams) {
            CUDA_TRY(cudaEventRecord(p->unload_fence, s), "lora_unload_adapter: fence");
            for (cudaStream_t ss : p->sides)
                CUDA_TRY(cudaStreamWaitEvent(ss, p->unload_fence, 0), "lora_unload_adapter: fence wait");
        }
        p->apply_streams.clear();
        if (it->second.ready) {
            // the load itself must also be finished before its pages are rewritten by a later load on
            // any side stream
            if (!it->second.ready_known)
                for (cudaStream_t ss : p->sides)
                    CUDA_TRY(cudaStreamWaitEvent(ss, (cudaEvent_t)it->second.ready, 0), "lora_unload_adapter: load wait");
            cudaEventDestroy((cudaEvent_t)it->second.ready);
        }
    }
    for (int pg : it->second.pages) p->page_used[pg] = 0;
    p->free_pages += it->second.rank;
    p->table.erase(it);
    ++p->table_version;
    return LORA_OK;
}

lora_status lora_adapter_ready(lora_pool* p, int32_t id, int* ready) {
    if (!p || !ready) return fail(LORA_ERR_ARG, "pool/ready is NULL");
    auto it = p->table.find(id);
    if (it == p->table.end()) return fail(LORA_ERR_UNKNOWN_ADAPTER, "adapter " + std::to_string(id) + " is not loaded");
    AdapterRec& a = it->second;
    if (!a.ready_known) {
        DeviceGuard g(p->device);
        cudaError_t e = cudaEventQuery((cudaEvent_t)a.ready);
        if (e == cudaSuccess) a.ready_known = true;
        else if (e != cudaErrorNotReady) return cuda_fail(e, "lora_adapter_ready");
        else cudaGetLastError();
    }
    *ready = a.ready_known ? 1 : 0;
    return LORA_OK;
}

lora_status lora_plan(lora_pool* p, const int32_t* seg_indptr, const int32_t* adapter_ids, int num_segments) {
    if (!p) return fail(LORA_ERR_ARG, "pool is NULL");
    std::string err;
    const bool tc = !p->host_only ? p->tc_prefill : prefill_supported(p->H_in, p->H_out, p->esz);
    lora_status s = build_plan(p->plan, seg_indptr, adapter_ids, num_segments, p->H_in, p->H_out, p->esz,
                               p->L_tc, tc, p->table, err, p->pad_max_rank ? p->n_pages : -1, p->num_sms);
    plan_uncached(p);
    if (s != LORA_OK) return fail(s, err);
    return LORA_OK;
}

// mode 0: full apply; 1: shrink only (partial v -> v_ext); 2: expand only (v_ext -> y, plan of the
// last shrink).  Modes 1/2 serve tensor parallelism: the caller all-reduces v in between.
static lora_status apply_impl(lora_pool* p, const void* x, void* y, const int32_t* seg_indptr,
                              const int32_t* adapter_ids, int num_segments, void* stream_ptr, int mode, float* v_ext,
                              int64_t v_cap, int64_t x_ld = 0, int64_t y_ld = 0) {
    if (!p) return fail(LORA_ERR_ARG, "pool is NULL");
    if (p->host_only) return fail(LORA_ERR_UNSUPPORTED, "apply on a host-only pool");
    lora_status s = LORA_OK;
    int T = 0;
    if (mode != 2) {
        if (num_segments < 0) return fail(LORA_ERR_ARG, "num_segments < 0");
        if (num_segments == 0) {
            p->split_ready = mode == 1;
            p->plan = Plan();
            plan_uncached(p);
            return LORA_OK;
        }
        if (!seg_indptr || !adapter_ids) return fail(LORA_ERR_ARG, "seg_indptr/adapter_ids is NULL");
        T = seg_indptr[num_segments];
        if (T == 0) {
            std::string err;
            s = build_plan(p->plan, seg_indptr, adapter_ids, num_segments, p->H_in, p->H_out, p->esz, p->L_tc, false,
                           p->table, err);
            plan_uncached(p);
            p->split_ready = (s == LORA_OK && mode == 1);
            return s == LORA_OK ? LORA_OK : fail(s, err);
        }
        if (!x) return fail(LORA_ERR_ARG, "x is NULL");
        if (((uintptr_t)x & 15)) return fail(LORA_ERR_ALIGN, "x must be 16-byte aligned");
    } else {
        if (!p->split_ready) return fail(LORA_ERR_ARG, "lora_apply_expand without a preceding lora_apply_shrink");
        T = p->plan.T;
        if (T == 0 || p->plan.n_gc == 0) {
            p->split_ready = false;
            return LORA_OK;
        }
    }
    if (mode != 1) {
        if (!y) return fail(LORA_ERR_ARG, "y is NULL");
        if (((uintptr_t)y & 15)) return fail(LORA_ERR_ALIGN, "y must be 16-byte aligned");
    }
    if (mode == 0) {
        const char* xs = (const char*)x;
        const char* ys = (const char*)y;
        const size_t xb = (size_t)T * p->H_in * p->esz, yb = (size_t)T * p->H_out * p->esz;
        if (xs < ys + yb && ys < xs + xb) return fail(LORA_ERR_ARG, "x and y overlap");
    }
    if (mode != 0 && !v_ext) return fail(LORA_ERR_ARG, "v buffer is NULL");
    if (mode != 0 && ((uintptr_t)v_ext & 3)) return fail(LORA_ERR_ALIGN, "v buffer must be 4-byte aligned");
    DeviceGuard g(p->device);
    cudaStream_t st = (cudaStream_t)stream_ptr;
    {
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return cuda_fail(e, "lora_apply: pending CUDA error");
    }
    if (mode != 2) {
        std::string err;
        const bool tc = p->tc_prefill && mode == 0;   // the split path keeps every token on the decode kernels
        s = plan_cached(p, seg_indptr, adapter_ids, num_segments, tc, p->pad_max_rank ? p->n_pages : -1, 0, err);
        if (s != LORA_OK) return fail(s, err);
        if (mode == 1 && p->plan.vred_floats > v_cap)
            return fail(LORA_ERR_ARG, "v buffer too small: need " + std::to_string(p->plan.vred_floats) + " floats");
        p->split_ready = false;
    }
    const Plan& pl = p->plan;
    if (mode == 1) p->split_ready = true;
    if (pl.G == 0) return LORA_OK;
    if (pl.n_gc == 0 && pl.n_pf_tiles == 0) return LORA_OK;
    if (mode == 2) p->split_ready = false;

    // order after in-flight loads of the adapters this batch reads
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    CUDA_TRY(cudaStreamIsCapturing(st, &cap), "lora_apply: capture query");
    p->capturing = cap != cudaStreamCaptureStatusNone;
    if (p->ready_gen != p->plan_gen) {   // (every adapter of an unchanged plan stays loaded)
        bool all = true;
        for (int gi = 0; gi < pl.G; ++gi) {
            AdapterRec& a = p->table.at(pl.group_id[gi]);
            if ((s = wait_loaded(a, st, p->capturing, "lora_apply: wait load")) != LORA_OK) return s;
            all = all && a.ready_known;
        }
        if (all) p->ready_gen = p->plan_gen;
    }
    // scratch (the k-slice partials live in the pool; the TP split's compact v is the caller's)
    if (pl.n_gc > 0 && mode != 2) {
        if ((s = grow(p, p->vbuf, p->vbuf_cap, (size_t)std::max<int64_t>(pl.vbuf_floats, 1), false, "vbuf")) != LORA_OK) return s;
    }
    if (pl.n_gc > 0 && mode == 1) {
        if ((s = grow(p, p->gc_cnt, p->gc_cnt_cap, (size_t)pl.n_gc, true, "gc_cnt")) != LORA_OK) return s;
    }
    if (pl.n_gc > 0 && mode != 2) {
        if ((s = grow(p, p->meta_dev, p->meta_cap, pl.blob.size(), false, "meta")) != LORA_OK) return s;
    }
    int launches = 0;
    if (pl.n_gc > 0) {
        DecodeLaunch L{x, y, p->dA, p->dB, p->vbuf, p->meta_dev, p->trace, p->H_in, p->H_out, p->esz, p->num_sms};
        L.phases = mode == 0 ? 3 : mode;
        L.vred = mode == 0 ? nullptr : v_ext;
        L.gc_cnt = mode == 1 ? p->gc_cnt : nullptr;
        L.x_ld = x_ld;
        L.y_ld = y_ld;
        cudaError_t e = (cudaError_t)launch_decode(pl, L, st, &launches);
        if (e != cudaSuccess) return cuda_fail(e, "lora_apply: decode kernel launch");
    }
    if (pl.n_pf_tiles > 0 && mode == 0) {
        if (pl.pf_cs > 1 &&
            (s = grow(p, p->pf_scratch, p->pf_scratch_cap, (size_t)pl.n_pf_tiles * 128 * kPfMaxRank, false, "pf_scratch")) != LORA_OK)
            return s;
        PrefillLaunch L{x, y, p->tm_a, p->tm_b, p->box_maps, nullptr, p->trace, T, p->H_in, p->H_out, p->n_pages, p->num_sms};
        L.pscratch = p->pf_scratch;
        cudaError_t e = (cudaError_t)launch_prefill(pl, L, st, &launches);
        if (e != cudaSuccess) return cuda_fail(e, "lora_apply: prefill kernel launch");
    }
    p->launches += launches;
    if (std::find(p->apply_streams.begin(), p->apply_streams.end(), st) == p->apply_streams.end())
        p->apply_streams.push_back(st);
    return LORA_OK;
}

lora_status lora_apply(lora_pool* p, const void* x, void* y, const int32_t* seg_indptr, const int32_t* adapter_ids,
                       int num_segments, void* stream) {
    return apply_impl(p, x, y, seg_indptr, adapter_ids, num_segments, stream, 0, nullptr, 0);
}

lora_status lora_apply_multi(lora_pool* const* pools, const void* const* xs, void* const* ys, int n_pools,
                             const int32_t* seg_indptr, const int32_t* adapter_ids, int num_segments, void* stream) {
    if (!pools || !xs || !ys) return fail(LORA_ERR_ARG, "pools/xs/ys is NULL");
    if (n_pools < 1 || n_pools > kMaxJobs) return fail(LORA_ERR_ARG, "n_pools must be in [1, 4]");
    if (n_pools == 1) return lora_apply(pools[0], xs[0], ys[0], seg_indptr, adapter_ids, num_segments, stream);
    lora_pool* p0 = pools[0];
    for (int i = 0; i < n_pools; ++i) {
        lora_pool* p = pools[i];
        if (!p) return fail(LORA_ERR_ARG, "pools[" + std::to_string(i) + "] is NULL");
        if (p->host_only) return fail(LORA_ERR_UNSUPPORTED, "apply on a host-only pool");
        if (p->device != p0->device || p->esz != p0->esz)
            return fail(LORA_ERR_ARG, "fused pools must share device and dtype");
        for (int j = 0; j < i; ++j)
            if (pools[j] == p) return fail(LORA_ERR_ARG, "a pool appears twice in one fused apply");
        if (!xs[i] || !ys[i]) return fail(LORA_ERR_ARG, "x/y of pool " + std::to_string(i) + " is NULL");
        if (((uintptr_t)xs[i] & 15) || ((uintptr_t)ys[i] & 15)) return fail(LORA_ERR_ALIGN, "x and y must be 16-byte aligned");
    }
    if (num_segments < 0) return fail(LORA_ERR_ARG, "num_segments < 0");
    if (num_segments == 0) return LORA_OK;
    if (!seg_indptr || !adapter_ids) return fail(LORA_ERR_ARG, "seg_indptr/adapter_ids is NULL");
    const int T = seg_indptr[num_segments];
    DeviceGuard g(p0->device);
    cudaStream_t st = (cudaStream_t)stream;
    {
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return cuda_fail(e, "lora_apply_multi: pending CUDA error");
    }
    // plans first (all validation before any launch: a failed call has no side effects)
    std::string err;
    for (int i = 0; i < n_pools; ++i) {
        lora_pool* p = pools[i];
        lora_status s = plan_cached(p, seg_indptr, adapter_ids, num_segments, p->tc_prefill, -1,
                                    n_pools > 1 ? kExpandSmemBudget : 0, err);
        if (s != LORA_OK) return fail(s, "pool " + std::to_string(i) + ": " + err);
        p->split_ready = false;
    }
    if (T == 0) return LORA_OK;
    lora_pool::FusedKey& fk = p0->fkey;
    bool same = fk.n == n_pools;
    for (int i = 0; same && i < n_pools; ++i) same = fk.pools[i] == pools[i] && fk.gens[i] == pools[i]->plan_gen;
    if (!same) {
        const Plan* parts[kMaxJobs];
        for (int i = 0; i < n_pools; ++i) parts[i] = &pools[i]->plan;
        fk.n = 0;
        lora_status s = merge_plans(parts, n_pools, p0->fused, err);
        if (s != LORA_OK) return fail(s, err);
        fk.n = n_pools;
        for (int i = 0; i < n_pools; ++i) { fk.pools[i] = pools[i]; fk.gens[i] = pools[i]->plan_gen; }
    }
    lora_status s = LORA_OK;
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    CUDA_TRY(cudaStreamIsCapturing(st, &cap), "lora_apply_multi: capture query");
    for (int i = 0; i < n_pools; ++i) pools[i]->capturing = cap != cudaStreamCaptureStatusNone;
    for (int i = 0; i < n_pools; ++i) {
        lora_pool* p = pools[i];
        if (p->ready_gen == p->plan_gen) continue;   // every adapter of an unchanged plan stays loaded
        bool all = true;
        for (int gi = 0; gi < p->plan.G; ++gi) {
            AdapterRec& a = p->table.at(p->plan.group_id[gi]);
            if ((s = wait_loaded(a, st, cap != cudaStreamCaptureStatusNone, "lora_apply_multi: wait load")) != LORA_OK)
                return s;
            all = all && a.ready_known;
        }
        if (all) p->ready_gen = p->plan_gen;
    }
    Plan& fz = p0->fused;
    int launches = 0;
    if (fz.n_gc > 0) {
        if ((s = grow(p0, p0->vbuf, p0->vbuf_cap, (size_t)std::max<int64_t>(fz.vbuf_floats, 1), false, "vbuf")) != LORA_OK) return s;
        if ((s = grow(p0, p0->meta_dev, p0->meta_cap, fz.blob.size(), false, "meta")) != LORA_OK) return s;
        DecodeLaunch L{xs[0], ys[0], p0->dA, p0->dB, p0->vbuf, p0->meta_dev, p0->trace, p0->H_in, p0->H_out, p0->esz,
                       p0->num_sms};
        L.n_jobs = n_pools;
        for (int i = 1; i < n_pools; ++i)
            L.more[i - 1] = DecodeLaunch::More{xs[i], ys[i], pools[i]->dA, pools[i]->dB, pools[i]->H_in, pools[i]->H_out};
        cudaError_t e = (cudaError_t)launch_decode(fz, L, st, &launches);
        if (e != cudaSuccess) return cuda_fail(e, "lora_apply_multi: decode kernel launch");
    }
    for (int i = 0; i < n_pools; ++i) {
        lora_pool* p = pools[i];
        if (p->plan.n_pf_tiles == 0) continue;
        if (p->plan.pf_cs > 1 &&
            (s = grow(p, p->pf_scratch, p->pf_scratch_cap, (size_t)p->plan.n_pf_tiles * 128 * kPfMaxRank, false, "pf_scratch")) !=
                LORA_OK)
            return s;
        PrefillLaunch L{xs[i], ys[i], p->tm_a, p->tm_b, p->box_maps, nullptr, p->trace, T, p->H_in, p->H_out, p->n_pages,
                        p->num_sms};
        L.pscratch = p->pf_scratch;
        cudaError_t e = (cudaError_t)launch_prefill(p->plan, L, st, &launches);
        if (e != cudaSuccess) return cuda_fail(e, "lora_apply_multi: prefill kernel launch");
    }
    p0->launches += launches;
    for (int i = 0; i < n_pools; ++i)
        if (std::find(pools[i]->apply_streams.begin(), pools[i]->apply_streams.end(), st) == pools[i]->apply_streams.end())
            pools[i]->apply_streams.push_back(st);
    return LORA_OK;
}

lora_status lora_apply_shrink(lora_pool* p, const void* x, const int32_t* seg_indptr, const int32_t* adapter_ids,
                              int num_segments, float* v_out, int64_t v_capacity, void* stream) {
    return apply_impl(p, x, nullptr, seg_indptr, adapter_ids, num_segments, stream, 1, v_out, v_capacity);
}

lora_status lora_apply_expand(lora_pool* p, void* y, const float* v_in, void* stream) {
    return apply_impl(p, nullptr, y, nullptr, nullptr, 0, stream, 2, const_cast<float*>(v_in), 0);
}

lora_status lora_tp_unique_id(void* id_out) {
    if (!id_out) return fail(LORA_ERR_ARG, "id_out is NULL");
    std::string err;
    const NcclApi* n = nccl(err);
    if (!n) return fail(LORA_ERR_NCCL, err);
    nccl_uid id;
    const int r = n->get_unique_id(&id);
    if (r != 0) return fail(LORA_ERR_NCCL, std::string("ncclGetUniqueId: ") + n->error_string(r));
    std::memcpy(id_out, &id, sizeof(id));
    return LORA_OK;
}

lora_status lora_tp_comm_create(const void* id, int tp_rank, int tp_size, lora_tp_comm** out) {
    if (!id || !out) return fail(LORA_ERR_ARG, "id/out is NULL");
    *out = nullptr;
    if (tp_size < 1 || tp_rank < 0 || tp_rank >= tp_size) return fail(LORA_ERR_ARG, "need 0 <= tp_rank < tp_size");
    std::string err;
    const NcclApi* n = nccl(err);
    if (!n) return fail(LORA_ERR_NCCL, err);
    lora_tp_comm* c = new lora_tp_comm();
    c->rank = tp_rank;
    c->size = tp_size;
    cudaGetDevice(&c->device);
    nccl_uid uid;
    std::memcpy(&uid, id, sizeof(uid));
    const int r = n->comm_init_rank(&c->comm, tp_size, uid, tp_rank);
    if (r != 0) {
        delete c;
        return fail(LORA_ERR_NCCL, std::string("ncclCommInitRank: ") + n->error_string(r));
    }
    *out = c;
    return LORA_OK;
}

lora_status lora_tp_comm_destroy(lora_tp_comm* c) {
    if (!c) return LORA_OK;
    std::string err;
    const NcclApi* n = nccl(err);
    int r = 0;
    if (n && c->comm) {
        DeviceGuard g(c->device);
        r = n->comm_destroy(c->comm);
    }
    delete c;
    if (r != 0) return fail(LORA_ERR_NCCL, std::string("ncclCommDestroy: ") + n->error_string(r));
    return LORA_OK;
}

lora_status lora_tp_init(lora_pool* p, lora_tp_comm* comm) {
    if (!p) return fail(LORA_ERR_ARG, "pool is NULL");
    if (p->host_only) return fail(LORA_ERR_UNSUPPORTED, "tensor parallelism on a host-only pool");
    if (comm && comm->device != p->device) return fail(LORA_ERR_ARG, "communicator and pool are on different devices");
    p->tp = comm;
    return LORA_OK;
}

lora_status lora_apply_tp(lora_pool* p, const void* x, int64_t x_ld, void* y, int64_t y_ld, const int32_t* seg_indptr,
                          const int32_t* adapter_ids, int num_segments, void* stream) {
    if (!p) return fail(LORA_ERR_ARG, "pool is NULL");
    if (!p->tp) return fail(LORA_ERR_ARG, "lora_apply_tp needs lora_tp_init");
    if (x_ld < 0 || y_ld < 0 || (x_ld && x_ld < p->H_in) || (y_ld && y_ld < p->H_out))
        return fail(LORA_ERR_ARG, "x_ld / y_ld must be 0 or at least hidden_in / hidden_out");
    if ((x_ld * p->esz) % 16 || (y_ld * p->esz) % 16) return fail(LORA_ERR_ALIGN, "x_ld / y_ld rows must be 16-B aligned");
    std::string err;
    const NcclApi* n = nccl(err);
    if (!n) return fail(LORA_ERR_NCCL, err);
    if (!y) return fail(LORA_ERR_ARG, "y is NULL");
    if (((uintptr_t)y & 15)) return fail(LORA_ERR_ALIGN, "y must be 16-byte aligned");
    // the compact v: planned first (every token on the decode kernels, as the split runs it) so its
    // buffer can be sized before anything is enqueued
    lora_status s = build_plan(p->plan, seg_indptr, adapter_ids, num_segments, p->H_in, p->H_out, p->esz, p->L_tc, false,
                               p->table, err);
    plan_uncached(p);
    if (s != LORA_OK) return fail(s, err);
    const size_t nv = (size_t)std::max<int64_t>(p->plan.vred_floats, 1);
    {
        DeviceGuard g(p->device);
        cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
        CUDA_TRY(cudaStreamIsCapturing((cudaStream_t)stream, &cap), "lora_apply_tp: capture query");
        p->capturing = cap != cudaStreamCaptureStatusNone;
        if ((s = grow(p, p->vred, p->vred_cap, nv, false, "vred")) != LORA_OK) return s;
    }
    s = apply_impl(p, x, nullptr, seg_indptr, adapter_ids, num_segments, stream, 1, p->vred, (int64_t)p->vred_cap, x_ld, 0);
    if (s != LORA_OK) return s;
    if (!p->split_ready || p->plan.n_gc == 0) {   // nothing to reduce or expand
        p->split_ready = false;
        return LORA_OK;
    }
    {
        DeviceGuard g(p->device);
        const int r = n->all_reduce(p->vred, p->vred, (size_t)p->plan.vred_floats, kNcclFloat32, kNcclSum, p->tp->comm,
                                    (cudaStream_t)stream);
        if (r != 0) {
            p->split_ready = false;
            return fail(LORA_ERR_NCCL, std::string("ncclAllReduce: ") + n->error_string(r));
        }
    }
    return apply_impl(p, nullptr, y, nullptr, nullptr, 0, stream, 2, p->vred, 0, 0, y_ld);
}

lora_status lora_apply_fused_base(lora_pool* p, const void* x, const void* W, void* y, const int32_t* seg_indptr,
                                  const int32_t* adapter_ids, int num_segments, void* stream) {
    if (!p) return fail(LORA_ERR_ARG, "pool is NULL");
    if (p->host_only) return fail(LORA_ERR_UNSUPPORTED, "apply on a host-only pool");
    if (p->esz != 2 || !p->tc_prefill || p->H_in % 64 || p->H_out % 128)
        return fail(LORA_ERR_UNSUPPORTED,
                    "the fused base GEMM needs a bf16 pool with hidden_in % 64 == 0 and hidden_out % 128 == 0");
    if (num_segments < 0) return fail(LORA_ERR_ARG, "num_segments < 0");
    if (num_segments == 0) return LORA_OK;
    if (!seg_indptr || !adapter_ids) return fail(LORA_ERR_ARG, "seg_indptr/adapter_ids is NULL");
    if (!x || !W || !y) return fail(LORA_ERR_ARG, "x/W/y is NULL");
    if (((uintptr_t)x & 15) || ((uintptr_t)W & 15) || ((uintptr_t)y & 15))
        return fail(LORA_ERR_ALIGN, "x, W and y must be 16-byte aligned");
    // validates the CSR and the ids into a scratch plan: the pool's own plan (the canonical metadata
    // of the last lora_apply, and a pending lora_apply_shrink's work) is left untouched
    std::string err;
    static thread_local Plan check;
    lora_status s = build_plan(check, seg_indptr, adapter_ids, num_segments, p->H_in, p->H_out, p->esz, p->L_tc, false,
                               p->table, err);
    if (s != LORA_OK) return fail(s, err);
    const int T = seg_indptr[num_segments];
    if (T == 0) return LORA_OK;
    {
        const char *xs = (const char*)x, *ws = (const char*)W, *ys = (const char*)y;
        const size_t xb = (size_t)T * p->H_in * 2, wb = (size_t)p->H_in * p->H_out * 2, yb = (size_t)T * p->H_out * 2;
        if ((xs < ys + yb && ys < xs + xb) || (ws < ys + yb && ys < ws + wb)) return fail(LORA_ERR_ARG, "y overlaps x or W");
    }
    // One launch (fused_base_kernel.cu): the GEMM y = [x | V]·[W ; B] over pairs of 128-token tiles of
    // one segment (an odd last tile runs alone), K extended by the adapter's rank; V = bf16(s·x·A) is
    // computed inside it by each adapter pair's first column tile (the "V items") into tile-private
    // rows of the pool's V scratch.  Pairs with an adapter come first (the kernel schedules their V
    // items first).
    if (p->H_out % 256)
        return fail(LORA_ERR_UNSUPPORTED, "the fused base GEMM needs hidden_out % 256 == 0");
    static thread_local std::vector<int32_t> words;              // pair records, then page lists
    static thread_local std::vector<int32_t> plain;              // pairs without an adapter (appended last)
    static thread_local std::vector<std::pair<int32_t, int32_t>> offs;   // (id, page offset in words)
    int n_pairs = 0, n_vtiles = 0, max_rp = 0, n_vp = 0;
    for (int i = 0; i < num_segments; ++i) {
        const int len = seg_indptr[i + 1] - seg_indptr[i];
        if (len <= 0) continue;
        n_pairs += (len + 255) / 256;
        if (adapter_ids[i] >= 0) {
            const AdapterRec& a = p->table.at(adapter_ids[i]);
            if (a.rank > kFusedMaxRank) return fail(LORA_ERR_UNSUPPORTED, "the fused base GEMM supports rank <= 128");
            n_vtiles += (len + 127) / 128;
            n_vp += (len + 255) / 256;
            max_rp = std::max(max_rp, (a.rank + 15) & ~15);
        }
    }
    words.assign((size_t)n_pairs * 10, 0);
    plain.clear();
    offs.clear();
    int pix = 0, vix = 0;
    for (int i = 0; i < num_segments; ++i) {
        const int len = seg_indptr[i + 1] - seg_indptr[i];
        if (len <= 0) continue;
        const int32_t id = adapter_ids[i];
        int rank = 0, off = 0;
        int32_t sb = 0;
        if (id >= 0) {
            const AdapterRec& a = p->table.at(id);
            rank = a.rank;
            std::memcpy(&sb, &a.scale, 4);
            off = -1;
            for (const auto& o : offs)
                if (o.first == id) off = o.second;
            if (off < 0) {
                off = (int)words.size();
                offs.emplace_back(id, off);
                words.insert(words.end(), a.pages.begin(), a.pages.end());
            }
        }
        int first_page = -1;   // the adapter's pages as one run: 2D box loads of its rank rows
        if (rank > 0) {
            const AdapterRec& a = p->table.at(id);
            bool run = true;
            for (int j = 1; j < rank && run; ++j) run = a.pages[j] == a.pages[0] + j;
            first_page = run ? a.pages[0] : -1;
        }
        for (int t0 = 0; t0 < len; t0 += 256) {
            int32_t rec[10];
            rec[0] = rank > 0 ? vix + t0 / 128 : 0;
            rec[1] = seg_indptr[i] + t0;
            rec[2] = std::min(128, len - t0);
            rec[3] = len - t0 > 128 ? seg_indptr[i] + t0 + 128 : 0;
            rec[4] = len - t0 > 128 ? std::min(128, len - t0 - 128) : 0;
            rec[5] = rank;
            rec[6] = off;
            rec[7] = sb;
            rec[8] = first_page;
            rec[9] = 0;
            if (rank > 0) {
                std::copy(rec, rec + 10, words.begin() + (size_t)pix * 10);
                ++pix;
            } else {
                plain.insert(plain.end(), rec, rec + 10);
            }
        }
        if (rank > 0) vix += (len + 127) / 128;
    }
    std::copy(plain.begin(), plain.end(), words.begin() + (size_t)pix * 10);
    if ((int)words.size() > kFusedBaseMaxWords)
        return fail(LORA_ERR_UNSUPPORTED, "batch too large for one fused launch (tiles and page lists exceed " +
                                              std::to_string(kFusedBaseMaxWords) + " words)");
    DeviceGuard g(p->device);
    cudaStream_t st = (cudaStream_t)stream;
    {
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return cuda_fail(e, "lora_apply_fused_base: pending CUDA error");
    }
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    CUDA_TRY(cudaStreamIsCapturing(st, &cap), "lora_apply_fused_base: capture query");
    p->capturing = cap != cudaStreamCaptureStatusNone;
    for (const auto& o : offs)
        if ((s = wait_loaded(p->table.at(o.first), st, p->capturing, "lora_apply_fused_base: wait load")) != LORA_OK)
            return s;
    const int v_cols = max_rp > 64 ? 128 : 64;
    int launches = 0;
    if (n_vtiles > 0) {
        if ((s = grow(p, p->fb_vtiles, p->fb_vtiles_cap, (size_t)n_vtiles * 128 * v_cols, false, "fused V tiles")) != LORA_OK)
            return s;
        if ((s = grow(p, p->fb_vsync, p->fb_vsync_cap, (size_t)n_vtiles + 2, true, "fused V sync")) != LORA_OK) return s;
    }
    FusedBaseLaunch L{x, W, y, p->tm_a, p->tm_b, T, p->H_in, p->H_out, p->n_pages};
    L.box_maps = p->box_maps;
    L.vtiles = n_vtiles > 0 ? p->fb_vtiles : nullptr;
    L.vsync = n_vtiles > 0 ? p->fb_vsync : nullptr;
    L.n_vtiles = n_vtiles;
    L.v_cols = v_cols;
    L.n_vp = n_vp;
    L.trace = p->trace;
    cudaError_t e = (cudaError_t)launch_fused_base(L, words.data(), (int)words.size(), n_pairs, p->num_sms, st);
    if (e != cudaSuccess) return cuda_fail(e, "lora_apply_fused_base: kernel launch");
    launches += 1;
    p->launches += launches;
    if (std::find(p->apply_streams.begin(), p->apply_streams.end(), st) == p->apply_streams.end())
        p->apply_streams.push_back(st);
    return LORA_OK;
}

lora_status lora_set_option(lora_pool* p, int option, int64_t value) {
    if (!p) return fail(LORA_ERR_ARG, "pool is NULL");
    ++p->table_version;   // planner settings may change: the cached plan is stale
    switch (option) {
        case LORA_OPT_TC_THRESHOLD:
            if (value < 1 || value > INT32_MAX) return fail(LORA_ERR_ARG, "L_tc must be >= 1");
            p->L_tc = (int)value;
            return LORA_OK;
        case LORA_OPT_RESERVE_TOKENS: {
            if (value < 0) return fail(LORA_ERR_ARG, "reserve must be >= 0");
            if (p->host_only) return LORA_OK;
            DeviceGuard g(p->device);
            p->capturing = false;   // a host call, not stream-ordered
            const int64_t ks = ksplit_of(p->H_in, p->esz);
            lora_status s = grow(p, p->vbuf, p->vbuf_cap, (size_t)std::max<int64_t>(1, value * ks * LORA_MAX_RANK), false, "vbuf");
            if (s == LORA_OK)
                s = grow(p, p->meta_dev, p->meta_cap, (size_t)(kHdrWords + (kGcFields + 1) * value + 4096), false, "meta");
            if (s == LORA_OK) s = grow(p, p->gc_cnt, p->gc_cnt_cap, (size_t)std::max<int64_t>(1, value), true, "gc_cnt");
            // prefill split-K partials: at most one 128 x 128 fp32 tile per CTA, and the planner keeps
            // split-K grids within the SM count
            const int64_t pf_ctas = std::min<int64_t>((value + 127) / 128 * 8, p->num_sms);
            if (s == LORA_OK && p->tc_prefill && value > 0)
                s = grow(p, p->pf_scratch, p->pf_scratch_cap, (size_t)pf_ctas * 128 * kPfMaxRank, false, "pf_scratch");
            return s;
        }
        case LORA_OPT_LOAD_KERNEL:
            if (value != 0 && value != 1) return fail(LORA_ERR_ARG, "LORA_OPT_LOAD_KERNEL takes 0 or 1");
            p->load_kernel = value == 1;
            return LORA_OK;
        case LORA_OPT_PAD_MAX_RANK:
            if (value != 0 && value != 1) return fail(LORA_ERR_ARG, "LORA_OPT_PAD_MAX_RANK takes 0 or 1");
            p->pad_max_rank = value == 1;
            return LORA_OK;
        default:
            return fail(LORA_ERR_ARG, "unknown option " + std::to_string(option));
    }
}

lora_status lora_pool_info(lora_pool* p, lora_pool_info_t* out) {
    if (!p || !out) return fail(LORA_ERR_ARG, "pool/out is NULL");
    std::memset(out, 0, sizeof(*out));
    out->hidden_in = p->H_in;
    out->hidden_out = p->H_out;
    out->max_adapters = p->max_adapters;
    out->max_total_rank = p->n_pages;
    out->dtype = (int32_t)p->dtype;
    out->elem_bytes = p->esz;
    out->resident_adapters = (int32_t)p->table.size();
    out->free_pages = p->free_pages;
    out->tc_threshold = p->L_tc;
    out->device = p->device;
    out->pool_bytes = (int64_t)p->n_pages * (p->H_in + p->H_out) * p->esz;
    int64_t rb = 0;
    for (auto& kv : p->table) rb += (int64_t)kv.second.rank * (p->H_in + p->H_out) * p->esz;
    out->resident_bytes = rb;
    out->kernel_launches = p->launches;
    return LORA_OK;
}

lora_status lora_debug_metadata(lora_pool* p, lora_metadata_view* o) {
    if (!p || !o) return fail(LORA_ERR_ARG, "pool/out is NULL");
    const Plan& pl = p->plan;
    std::memset(o, 0, sizeof(*o));
    o->T = pl.T; o->S = pl.S; o->G = pl.G; o->L_tc = pl.L_tc;
    o->tok_seg = pl.tok_seg.data();
    o->group_id = pl.group_id.data();
    o->group_rank = pl.group_rank.data();
    o->group_scale = pl.group_scale.data();
    o->group_ntok = pl.group_ntok.data();
    o->group_page_off = pl.group_page_off.data();
    o->group_tok_off = pl.group_tok_off.data();
    o->group_tokens = pl.group_tokens.data();
    o->pages = pl.pages.data();
    o->seg_kind = pl.seg_kind.data();
    o->n_seg = pl.n_seg; o->max_rank = pl.max_rank; o->nseg_x_maxrank = pl.nseg_x_maxrank;
    o->sum_rank_seg = pl.sum_rank_seg; o->sum_rank_groups = pl.sum_rank_groups; o->sum_rank_tokens = pl.sum_rank_tokens;
    o->n_decode_units = pl.n_shrink + pl.n_expand;
    o->n_shrink_units = pl.n_shrink;
    o->n_expand_units = pl.n_expand;
    o->v_floats = pl.vred_floats;
    o->n_prefill_tiles = pl.n_prefill_tiles;
    o->n_prefill_ctas = pl.n_pf_tiles;
    o->prefill_cluster = pl.pf_cs;
    return LORA_OK;
}

lora_status lora_debug_set_trace(lora_pool* p, void* dev_buf) {
    if (!p) return fail(LORA_ERR_ARG, "pool is NULL");
    p->trace = static_cast<unsigned long long*>(dev_buf);
    return LORA_OK;
}

lora_status lora_debug_adapter_pages(lora_pool* p, int32_t id, int32_t* pages, int cap, int* rank) {
    if (!p) return fail(LORA_ERR_ARG, "pool is NULL");
    auto it = p->table.find(id);
    if (it == p->table.end()) return fail(LORA_ERR_UNKNOWN_ADAPTER, "adapter " + std::to_string(id) + " is not loaded");
    if (rank) *rank = it->second.rank;
    if (pages)
        for (int j = 0; j < it->second.rank && j < cap; ++j) pages[j] = it->second.pages[j];
    return LORA_OK;
}

lora_status lora_debug_read_pages(lora_pool* p, int32_t id, void* A_out, void* B_out) {
    if (!p || !A_out || !B_out) return fail(LORA_ERR_ARG, "pool/A_out/B_out is NULL");
    if (p->host_only) return fail(LORA_ERR_UNSUPPORTED, "host-only pool has no device pages");
    auto it = p->table.find(id);
    if (it == p->table.end()) return fail(LORA_ERR_UNKNOWN_ADAPTER, "adapter " + std::to_string(id) + " is not loaded");
    DeviceGuard g(p->device);
    for (cudaStream_t ss : p->sides) CUDA_TRY(cudaStreamSynchronize(ss), "lora_debug_read_pages: sync");
    const size_t ra = (size_t)p->H_in * p->esz, rb = (size_t)p->H_out * p->esz;
    for (int j = 0; j < it->second.rank; ++j) {
        CUDA_TRY(cudaMemcpy((char*)A_out + j * ra, p->dA + (size_t)it->second.pages[j] * ra, ra, cudaMemcpyDeviceToHost), "read A");
        CUDA_TRY(cudaMemcpy((char*)B_out + j * rb, p->dB + (size_t)it->second.pages[j] * rb, rb, cudaMemcpyDeviceToHost), "read B");
    }
    return LORA_OK;
}

}  // extern "C"
