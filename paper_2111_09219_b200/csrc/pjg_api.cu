// C-ABI (include/pjg.h) and host orchestration of the fully-on-GPU decode.
//
// Host work per batch is the reference's header walk (parser.hpp:264-347
// minus the scan), Huffman/quant table setup (huffman.hpp:60-93) and the
// layout plan; then ONE H2D of the compressed bytes (plus one of a small
// descriptor blob) and six stream-ordered kernels (K0, K1, K1c, K2, K3, K4).
// No host synchronisation between kernels; no CPU fallback anywhere: if the
// device path fails the call fails.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <string>
#include <atomic>
#include <condition_variable>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

#include "../../include/pjg.h"
#include "devparse.h"
#include "jfif.hpp"
#include "pjg_internal.h"

using namespace pjg;

namespace {

constexpr uint32_t kNumEvents = PJG_NUM_STAGES + 1;

struct DevBuf {
    void* p = nullptr;
    size_t cap = 0;
    bool zero = false;  // zero-fill on (re)allocation (lookback flag arrays)
    cudaStream_t zs = nullptr;  // the owning context's stream: the fill is ordered before its kernels

    cudaError_t ensure(size_t n) {
        if (n <= cap && p) return cudaSuccess;
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
        size_t want = std::max<size_t>(n + n / 4, 256);
        cudaError_t e = cudaMalloc(&p, want);
        if (e != cudaSuccess) return e;
        cap = want;
        if (zero) e = cudaMemsetAsync(p, 0, want, zs);
        return e;
    }
    template <class T>
    T* as() const {
        return static_cast<T*>(p);
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
    }
};

struct HostBuf {  // pinned
    void* p = nullptr;
    size_t cap = 0;
    cudaError_t ensure(size_t n) {
        if (n <= cap && p) return cudaSuccess;
        if (p) cudaFreeHost(p);
        p = nullptr;
        cap = 0;
        size_t want = std::max<size_t>(n + n / 4, 4096);
        cudaError_t e = cudaMallocHost(&p, want);
        if (e == cudaSuccess) cap = want;
        return e;
    }
    void release() {
        if (p) cudaFreeHost(p);
        p = nullptr;
        cap = 0;
    }
};

size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

// Host worker threads of a context, started once: batch planning runs a few
// parallel passes per batch, and spawning threads for each cost more than the
// passes themselves on thumbnail batches.
class WorkerPool {
public:
    ~WorkerPool() {
        {
            std::lock_guard<std::mutex> g(m_);
            stop_ = true;
        }
        cv_.notify_all();
        for (auto& t : th_) t.join();
    }
    // fn(0..n-1), the calling thread taking part; returns when all are done
    void run(unsigned n, const std::function<void(unsigned)>& fn) {
        if (n <= 1) {
            if (n) fn(0);
            return;
        }
        start(n - 1);
        {
            std::lock_guard<std::mutex> g(m_);
            job_ = &fn;
            njobs_ = n;
            next_.store(0);
            pending_ = n;
            ++gen_;
        }
        cv_.notify_all();
        work();
        std::unique_lock<std::mutex> g(m_);
        done_.wait(g, [&] { return pending_ == 0; });
        job_ = nullptr;
    }

private:
    void start(unsigned want) {
        while (th_.size() < want) th_.emplace_back([this] { loop(); });
    }
    void work() {
        for (;;) {
            const unsigned i = next_.fetch_add(1);
            if (i >= njobs_) return;
            (*job_)(i);
            std::lock_guard<std::mutex> g(m_);
            if (--pending_ == 0) done_.notify_all();
        }
    }
    void loop() {
        uint64_t seen = 0;
        for (;;) {
            {
                std::unique_lock<std::mutex> g(m_);
                cv_.wait(g, [&] { return stop_ || gen_ != seen; });
                if (stop_) return;
                seen = gen_;
            }
            work();
        }
    }
    std::vector<std::thread> th_;
    std::mutex m_;
    std::condition_variable cv_, done_;
    const std::function<void(unsigned)>* job_ = nullptr;
    unsigned njobs_ = 0, pending_ = 0;
    std::atomic<unsigned> next_{0};
    uint64_t gen_ = 0;
    bool stop_ = false;
};

}  // namespace

struct pjg_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    std::string err;
    uint32_t epoch = 0;
    bool busy = false;
    double basis[64];
    cudaEvent_t ev[kNumEvents] = {};
    DevBuf raw, ubuf, meta, blkmeta, ent, dcs, off, cap, pred, cta_end, cta_start, k1_flag, coef, out, segs, sym, tag,
        counters, k0_flag, k0_agg, k2_flag, k2_agg, stats, plan, meta2, ents, umeta, eoff, k5tmp;
    HostBuf stage, meta_host, status_host, desc_host, plan_host;
    WorkerPool pool_threads;
    // Per-image host arrays, lent to the live batch and taken back at destroy:
    // thumbnail batches hold tens of thousands of images, and fresh vectors
    // would be mmap'd and page-faulted again on every batch.
    struct Scratch {
        std::vector<int32_t> host_status;
        std::vector<pjg_image_info> info;
        std::vector<ImgState> dev_state;
    } pool;
};

struct pjg_batch {
    pjg_ctx* ctx = nullptr;
    pjg_config cfg{};
    size_t n = 0;
    const ImgDesc* desc = nullptr;  // n descriptors in ctx->desc_host
    std::vector<int32_t> host_status;
    std::vector<pjg_image_info> info;
    // raw layout
    const uint8_t* raw_src = nullptr;  // contiguous user region, or ctx->stage
    size_t raw_bytes = 0;
    bool packed = false;
    // meta blob layout (offsets into ctx->meta)
    size_t m_dri = 0, m_desc = 0, m_state = 0, m_huff = 0, m_quant = 0, m_wq = 0, m_basis = 0, m_k0 = 0, m_tile = 0,
           m_sub = 0, m_k0img = 0, m_subimg = 0, m_total = 0;
    uint32_t n_huff = 0, n_quant = 0;
    uint32_t k0_tiles = 0, k4_tiles = 0, k1_ctas = 0, k2_tiles = 0;
    uint64_t total_subs = 0, total_dus = 0, out_bytes = 0, seg_total = 0;
    uint64_t sb_int = 0;  // internal subsequence size (divides cfg.subsequence_bits)
    Params prm{};
    bool uploaded = false, decoded = false, synced = false;
    // device-planned batch (pjg_batch_create_device): descriptors, statuses and
    // image infos live on the device; the host copies are fetched on first use
    bool devplan = false, host_view = false;
    const ImgState* state0 = nullptr;      // device: initial per-image statuses
    const pjg_image_info* dinfo = nullptr; // device: per-image infos
    cudaGraphExec_t gexec = nullptr;       // captured decode (latency-bound batches)
    std::vector<ImgState> dev_state;  // fetched at synchronize
    void swap_pool(pjg_ctx::Scratch& p) {
        host_status.swap(p.host_status);
        info.swap(p.info);
        dev_state.swap(p.dev_state);
    }
    double stage_ms[PJG_NUM_STAGES] = {};
    unsigned long long stats[kNumStats] = {};
};

namespace {

int fail(pjg_ctx* c, int code, const std::string& msg) {
    if (c) c->err = msg;
    return code;
}

int cuda_fail(pjg_ctx* c, cudaError_t e, const char* where) {
    return fail(c, PJG_CUDA_ERROR, std::string(where) + ": " + cudaGetErrorString(e));
}

#define CU(call, where)                                          \
    do {                                                         \
        cudaError_t e__ = (call);                                \
        if (e__ != cudaSuccess) return cuda_fail(ctx, e__, where); \
    } while (0)

uint64_t out_bytes_for(const Header& h, uint32_t mode) {
    if (h.comps.empty()) return 0;
    if (mode == PJG_OUT_RGB) return uint64_t(h.width) * h.height * (h.comps.size() == 3 ? 3 : 1);
    if (mode == PJG_OUT_GRAY) return uint64_t(h.comp_width(0)) * h.comp_height(0);
    uint64_t s = 0;
    for (size_t c = 0; c < h.comps.size(); ++c) s += uint64_t(h.comp_width(c)) * h.comp_height(c);
    return s;
}

void fill_info(const Header& h, uint32_t mode, size_t compressed, pjg_image_info* info) {
    std::memset(info, 0, sizeof(*info));
    info->compressed_bytes = compressed;
    if (h.status != kOk && h.comps.empty()) return;
    info->width = h.width;
    info->height = h.height;
    info->num_components = uint32_t(h.comps.size());
    for (size_t c = 0; c < h.comps.size() && c < 3; ++c) {
        info->plane_width[c] = h.comp_width(c);
        info->plane_height[c] = h.comp_height(c);
    }
    info->h_max = h.h_max;
    info->v_max = h.v_max;
    info->mcus_x = h.mcus_x;
    info->mcus_y = h.mcus_y;
    info->data_units = h.total_dus();
    info->channels = mode == PJG_OUT_RGB ? (h.comps.size() == 3 ? 3 : 1)
                                         : (mode == PJG_OUT_GRAY ? 1 : uint32_t(h.comps.size()));
    info->output_bytes = out_bytes_for(h, mode);
}

bool validate_cfg(pjg_ctx* ctx, const pjg_config* cfg, int* st) {
    // partition() validation (parallel_decode.hpp:50-62)
    if (!cfg || cfg->subsequence_bits == 0 || cfg->subsequence_bits % 32 != 0 ||
        cfg->sequence_length_b == 0) {
        *st = fail(ctx, PJG_CONSISTENCY_FAILURE,
                   "subsequence_bits must be a positive multiple of 32 and sequence_length_b >= 1");
        return false;
    }
    if (cfg->output > PJG_OUT_GRAY) {
        *st = fail(ctx, PJG_INVALID_ARGUMENT, "bad output kind");
        return false;
    }
    return true;
}

}  // namespace

// ====================================================================== API
extern "C" {

const char* pjg_status_name(int s) {
    switch (s) {
        case PJG_OK: return "Ok";
        case PJG_MALFORMED_STUFFING: return "MalformedStuffing";
        case PJG_EMPTY_SCAN: return "EmptyScan";
        case PJG_OUT_OF_BITS: return "OutOfBits";
        case PJG_UNSUPPORTED_FEATURE: return "UnsupportedFeature";
        case PJG_MALFORMED_HEADER: return "MalformedHeader";
        case PJG_MISSING_TABLE: return "MissingTable";
        case PJG_OVERSUBSCRIBED_CODE: return "OversubscribedCode";
        case PJG_INVALID_CODE: return "InvalidCode";
        case PJG_CONSISTENCY_FAILURE: return "ConsistencyFailure";
        case PJG_EMPTY_CORPUS: return "EmptyCorpus";
        case PJG_IO_ERROR: return "IoError";
        case PJG_CUDA_ERROR: return "CudaError";
        case PJG_INVALID_ARGUMENT: return "InvalidArgument";
        case PJG_CAPACITY: return "Capacity";
        case PJG_NOT_DECODED: return "NotDecoded";
    }
    return "Unknown";
}

void pjg_default_config(pjg_config* cfg) {
    cfg->subsequence_bits = 1024;
    cfg->sequence_length_b = 256;
    cfg->output = PJG_OUT_PLANES;
    cfg->restart_intervals = 0;
    cfg->reserved = 0;
}

int pjg_ctx_create(int device, pjg_ctx** out) {
    if (!out) return PJG_INVALID_ARGUMENT;
    *out = nullptr;
    auto c = std::make_unique<pjg_ctx>();
    pjg_ctx* ctx = c.get();
    c->device = device;
    CU(cudaSetDevice(device), "cudaSetDevice");
    CU(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking), "cudaStreamCreate");
    for (auto& e : c->ev) CU(cudaEventCreate(&e), "cudaEventCreate");
    c->k0_flag.zero = c->k2_flag.zero = c->k1_flag.zero = c->tag.zero = true;
    for (DevBuf* b : {&c->k0_flag, &c->k2_flag, &c->k1_flag, &c->tag}) b->zs = c->stream;
    // IdctBasis (transform.hpp:93-108): the same host libm expression.
    for (int u = 0; u < 8; ++u) {
        double cu = u == 0 ? 1.0 / std::sqrt(2.0) : 1.0;
        for (int x = 0; x < 8; ++x) c->basis[u * 8 + x] = 0.5 * cu * std::cos((2 * x + 1) * u * M_PI / 16.0);
    }
    *out = c.release();
    return PJG_OK;
}

void pjg_ctx_destroy(pjg_ctx* c) {
    if (!c) return;
    cudaSetDevice(c->device);
    if (c->stream) cudaStreamSynchronize(c->stream);
    for (DevBuf* b : {&c->raw, &c->ubuf, &c->meta, &c->blkmeta, &c->ent, &c->dcs, &c->off, &c->cap, &c->pred,
                      &c->cta_end, &c->cta_start, &c->k1_flag, &c->coef, &c->out, &c->counters,
                      &c->k0_flag, &c->k0_agg, &c->k2_flag, &c->k2_agg, &c->stats, &c->segs, &c->sym, &c->tag, &c->plan, &c->meta2,
                      &c->ents, &c->umeta, &c->eoff, &c->k5tmp})
        b->release();
    c->stage.release();
    c->meta_host.release();
    c->desc_host.release();
    c->status_host.release();
    c->plan_host.release();
    for (auto& e : c->ev)
        if (e) cudaEventDestroy(e);
    if (c->stream) cudaStreamDestroy(c->stream);
    delete c;
}

const char* pjg_last_error(const pjg_ctx* c) { return c ? c->err.c_str() : "null context"; }
void* pjg_ctx_stream(pjg_ctx* c) { return c ? (void*)c->stream : nullptr; }

int pjg_inspect(const uint8_t* file, size_t size, uint32_t output, pjg_image_info* info) {
    if (!file || !info) return PJG_INVALID_ARGUMENT;
    Header h = parse_header(file, size);
    fill_info(h, output, size, info);
    return h.status;
}

int pjg_inspect_header(const uint8_t* file, size_t size, int allow_dri, pjg_header_info* out) {
    if (!file || !out) return PJG_INVALID_ARGUMENT;
    std::memset(out, 0, sizeof(*out));
    const Header h = parse_header(file, size, allow_dri != 0);
    out->width = h.width;
    out->height = h.height;
    out->num_components = uint32_t(h.comps.size());
    for (size_t c = 0; c < h.comps.size() && c < 3; ++c) {
        out->comp_id[c] = h.comps[c].id;
        out->comp_h[c] = h.comps[c].h;
        out->comp_v[c] = h.comps[c].v;
        out->comp_tq[c] = h.comps[c].tq;
        out->comp_td[c] = h.comps[c].td;
        out->comp_ta[c] = h.comps[c].ta;
    }
    out->mcu_width = 8 * h.h_max;
    out->mcu_height = 8 * h.v_max;
    out->mcus_x = h.mcus_x;
    out->mcus_y = h.mcus_y;
    out->data_units_per_mcu = h.dpm;
    out->total_data_units = h.total_dus();
    for (int t = 0; t < 4; ++t) {
        out->quant_tables += h.quant_present[t] ? 1u : 0u;
        out->dc_tables += h.dc[t].present ? 1u : 0u;
        out->ac_tables += h.ac[t].present ? 1u : 0u;
    }
    out->restart_interval = h.restart_interval;
    out->scan_offset = h.scan_start;
    return h.status;
}

namespace {
// smallest internal subsequence size for small batches (PJG_SB_MIN overrides, A/B)
uint64_t sb_floor() {
    const char* e = getenv("PJG_SB_MIN");
    const long v = e ? atol(e) : 0;
    return (v >= 32 && v % 32 == 0) ? uint64_t(v) : 64u;  // cfg 1: 256 -> 64 bits: 0.19 -> 0.157 ms
}

// Internal subsequence size: halve sb while the batch would give K1 fewer than
// `target` subsequences (default: half the GPU's K1 threads at one CTA per SM;
// PJG_SB_TARGET overrides, PJG_SB_AUTO=0 disables).  Restart-interval batches
// keep sb (their per-interval partitions are dumped as is).
uint64_t internal_sb(uint64_t sb, uint64_t bits, bool allowed) {
    uint64_t sb_int = sb;
    const char* e = getenv("PJG_SB_AUTO");
    if (!allowed || (e && atoi(e) == 0)) return sb;
    uint64_t target = uint64_t(kK1Threads) * 148 / 2;
    if (const char* t = getenv("PJG_SB_TARGET")) target = std::max<long>(1, atol(t));
    uint64_t est = bits / sb;
    while (est < target && sb_int / 2 >= sb_floor() && (sb_int / 2) % 32 == 0) {
        sb_int /= 2;
        est *= 2;
    }
    return sb_int;
}

// Per-batch totals of a plan (host planner or devplan.cu) and where its
// device-side tables live: everything the buffer reservation and the kernel
// parameters need.
struct PlanSummary {
    size_t n = 0;
    uint64_t sub = 0, du = 0, outb = 0, seg_total = 0, bits = 0, n_ok = 0, sb = 0, sb_int = 0, max_du = 0;
    uint32_t k0t = 0, k4t = 0, ndri = 0, n_huff = 0, n_quant = 0, k0_bpt = 0;
    bool all420 = false;
};
struct MetaPtrs {
    uint8_t *desc, *state, *huff, *quant, *wq, *basis, *k0, *tile, *sub, *k0img, *subimg, *dri;
};

int finish_plan(pjg_ctx* ctx, pjg_batch* b, const PlanSummary& S, const MetaPtrs& M) {
    b->n_huff = S.n_huff;
    b->n_quant = S.n_quant;
    b->k0_tiles = S.k0t;
    b->k4_tiles = S.k4t;
    b->total_subs = S.sub;
    b->total_dus = S.du;
    b->seg_total = S.seg_total;
    b->out_bytes = S.outb;
    b->sb_int = S.sb_int;
    b->k1_ctas = uint32_t((S.sub + kK1Own - 1) / kK1Own);
    b->k2_tiles = uint32_t((S.sub + kK2Threads - 1) / kK2Threads);
    // ---- device reservation
    CU(ctx->raw.ensure(b->raw_bytes + 64), "cudaMalloc(raw)");
    CU(ctx->ubuf.ensure(b->raw_bytes + 64), "cudaMalloc(ubuf)");
    const size_t subs = std::max<uint64_t>(S.sub, 1);
    CU(ctx->ent.ensure(subs * sizeof(Entry)), "cudaMalloc(ent)");
    CU(ctx->dcs.ensure(subs * sizeof(DcSums)), "cudaMalloc(dcs)");
    CU(ctx->off.ensure(subs * 8), "cudaMalloc(off)");
    CU(ctx->cap.ensure(subs * 4), "cudaMalloc(cap)");
    CU(ctx->pred.ensure(subs * sizeof(DcSums)), "cudaMalloc(pred)");
    CU(ctx->cta_end.ensure((b->k1_ctas + 1) * sizeof(Entry)), "cudaMalloc(cta_end)");
    CU(ctx->cta_start.ensure((b->k1_ctas + 1) * sizeof(Entry)), "cudaMalloc(cta_start)");
    // K1 chains keep their decoded symbols for K3 to replay (16 bits each, up
    // to sb/4 per subsequence: 4 bytes of scratch per compressed byte) when it
    // pays: measured break-even — many symbols per data unit
    // (K3's decode dominates its block work) but a stream that syncs in few
    // rounds (K1 stores each chain's symbols once per round): 64..160 scan
    // bits per data unit, in images of >= 64 subsequences on average.
    // PJG_REPLAY=0/1 forces it.
    // small batches (under ~4 K1 CTAs per SM): the decoders' table probes sit on a
    // serial dependency chain with few warps to hide an L1 miss — stage the
    // tables in shared memory
    uint32_t smem_tables =
        (S.n_huff <= kMaxSmemTables && S.sub < uint64_t(kK1Threads) * 148 * 4) ? S.n_huff : 0u;
    if (const char* e = getenv("PJG_SMEM_TABLES"))  // override (A/B experiments)
        smem_tables = (atoi(e) && S.n_huff <= kMaxSmemTables) ? S.n_huff : 0u;
    const bool st_tables = smem_tables != 0;
    bool replay_on = false;
    {
        const uint64_t per_du = S.du ? S.bits / S.du : 0;
        // (and large images: a few subsequences per image keep K3 cheap)
        // (large batches only: K1's shared-memory-table variant for small ones
        // does not keep symbols)
        // (dense interface only: with the compact one K3 is cheap enough that
        // K1's symbol stores cost more than the replay saves — cfg 4: step 5.97
        // ms with replay, 5.60 without)
        replay_on = per_du > 128 && per_du <= 160 && S.n_ok && S.sub / S.n_ok >= 64 && !st_tables;
        if (const char* e = getenv("PJG_REPLAY")) replay_on = atoi(e) != 0 && !st_tables;
        if (getenv("PJG_NO_REPLAY")) replay_on = false;
    }
    const uint32_t sym_cap = (!replay_on || S.sb_int > 65536) ? 0u : uint32_t(S.sb_int / 4);
    const uint64_t sym_stride = align_up(subs, 64);
    if (sym_cap) {
        CU(ctx->sym.ensure(sym_stride * sym_cap * 2), "cudaMalloc(sym)");
        CU(ctx->tag.ensure(subs * 16), "cudaMalloc(tag)");
    }
    CU(ctx->k1_flag.ensure((b->k1_ctas + 1) * 4), "cudaMalloc(k1_flag)");
    CU(ctx->coef.ensure(std::max<uint64_t>(S.du, 1) * 128), "cudaMalloc(coef)");
    // Compact K3 -> K4 interface (Params::compact): per-subsequence entry counts
    // ride in 16 bits (sb <= 65535) and entry positions are image-relative 32-bit
    // (64 x the largest image's units < 2^32).  PJG_COMPACT=0 forces the dense
    // int16 coefficient buffer (A/B, parity).
    // Measured: compact wins while units are short enough — K3
    // drops its staging block, K4's per-entry scatter costs about what dense
    // column dequantisation does (cfg 3, 31 bits/unit: step -6 %; cfg 4, 83:
    // -4 %) — and loses on very long units (q100 4:4:4, 265 bits/unit: +10 %):
    // <= 128 scan bits per data unit.
    bool compact = S.sb_int <= 65535 && S.max_du * 64 < (1ull << 32) && S.du && S.bits <= 128 * S.du;
    if (const char* e = getenv("PJG_COMPACT")) compact = S.sb_int <= 65535 && S.max_du * 64 < (1ull << 32) && atoi(e) != 0;
    if (compact) {
        CU(ctx->ents.ensure(std::max<uint64_t>(S.du, 1) * 256), "cudaMalloc(ents)");
        CU(ctx->umeta.ensure(std::max<uint64_t>(S.du, 1) * 16), "cudaMalloc(umeta)");
        CU(ctx->eoff.ensure(subs * 4), "cudaMalloc(eoff)");
    }
    CU(ctx->segs.ensure(std::max<uint64_t>(S.seg_total, 1) * sizeof(uint2)), "cudaMalloc(segs)");
    CU(ctx->blkmeta.ensure(std::max<uint64_t>(S.du, 1) * 8), "cudaMalloc(blkmeta)");
    CU(ctx->out.ensure(std::max<uint64_t>(S.outb, 1)), "cudaMalloc(out)");
    CU(ctx->counters.ensure(kNumCounters * 4), "cudaMalloc(counters)");
    CU(ctx->stats.ensure(kNumStats * 8), "cudaMalloc(stats)");
    CU(ctx->k0_flag.ensure((S.k0t + 1) * 4), "cudaMalloc(k0_flag)");
    CU(ctx->k0_agg.ensure((S.k0t + 1) * 32), "cudaMalloc(k0_agg)");
    CU(ctx->k2_flag.ensure((b->k2_tiles + 1) * 4), "cudaMalloc(k2_flag)");
    CU(ctx->k2_agg.ensure((b->k2_tiles + 1) * 64), "cudaMalloc(k2_agg)");
    CU(ctx->status_host.ensure(S.n * sizeof(ImgState) + 64 + kNumStats * 8), "cudaMallocHost(status)");

    // ---- kernel parameters
    Params& p = b->prm;
    p.img = reinterpret_cast<const ImgDesc*>(M.desc);
    p.ist = reinterpret_cast<ImgState*>(M.state);
    p.n_img = uint32_t(S.n);
    p.huff = reinterpret_cast<const DevHuff*>(M.huff);
    p.quant_raster = reinterpret_cast<const uint16_t*>(M.quant);
    p.basis = reinterpret_cast<const double*>(M.basis);
    p.wq = reinterpret_cast<const float*>(M.wq);
    p.n_quant = S.n_quant;
    p.raw = ctx->raw.as<uint8_t>();
    p.ubuf = ctx->ubuf.as<uint8_t>();
    p.k0_first = reinterpret_cast<const uint32_t*>(M.k0);
    p.k0_img = reinterpret_cast<const uint32_t*>(M.k0img);
    p.sub_img = reinterpret_cast<const uint32_t*>(M.subimg);
    p.segs = ctx->segs.as<uint2>();
    p.dri_img = reinterpret_cast<const uint32_t*>(M.dri);
    p.n_dri = S.ndri;
    p.k0_tiles = S.k0t;
    p.k0_bpt = S.k0_bpt;
    p.smem_tables = smem_tables;
    p.k1_ctas = b->k1_ctas;
    p.n_huff = b->n_huff;
    // grids that do not fill the GPU are latency-bound: a stale CTA start is
    // re-chained inside K1 from shared memory; full grids skip the wait and
    // leave the (few) stale starts to K1c's parallel first pass
    p.k1_hop = b->k1_ctas < 2 * 148 ? 1u : 0u;
    if (const char* e = getenv("PJG_K1_HOP")) p.k1_hop = atoi(e) ? 1u : 0u;  // override (tests, A/B)
    {  // every image 4:2:0 colour to RGB: K4's specialised variant
        const bool all420 = S.all420 && b->cfg.output == PJG_OUT_RGB;
        p.k4_layout = all420 ? 1u : 0u;
        if (const char* e = getenv("PJG_K4_LAYOUT")) p.k4_layout = atoi(e) == 1 && all420 ? 1u : 0u;  // A/B
    }
    p.sb = S.sb_int;
    p.sb_cfg = S.sb;
    p.b_cfg = b->cfg.sequence_length_b;
    p.sub_first = reinterpret_cast<const uint64_t*>(M.sub);
    p.total_subs = S.sub;
    p.ent = ctx->ent.as<Entry>();
    p.dcs = ctx->dcs.as<DcSums>();
    p.off = ctx->off.as<uint64_t>();
    p.cap = ctx->cap.as<uint32_t>();
    p.pred = ctx->pred.as<DcSums>();
    p.cta_end = ctx->cta_end.as<Entry>();
    p.cta_start = ctx->cta_start.as<Entry>();
    p.sym = sym_cap ? ctx->sym.as<uint16_t>() : nullptr;
    p.tag = sym_cap ? ctx->tag.as<uint32_t>() : nullptr;
    p.sym_stride = sym_stride;
    p.sym_cap = sym_cap;
    p.k1_flag = ctx->k1_flag.as<uint32_t>();
    p.k2_tiles = b->k2_tiles;
    p.k4_tiles = S.k4t;
    p.tile_first = reinterpret_cast<const uint32_t*>(M.tile);
    p.coef = ctx->coef.as<int16_t>();
    p.meta = ctx->blkmeta.as<uint2>();
    p.compact = compact ? 1u : 0u;
    // K3's table probes sit on the decoder's serial chain: compact K3 (69
    // registers, no staging block) keeps 4 CTAs per SM even with the tables
    // in shared memory (cfg 3: 1.37 -> 1.27 ms); dense K3 loses occupancy
    p.k3_tables = (compact && S.n_huff <= kMaxSmemTables) ? S.n_huff : smem_tables;
    if (const char* e = getenv("PJG_K3_TABLES")) p.k3_tables = (atoi(e) && S.n_huff <= kMaxSmemTables) ? S.n_huff : 0u;
    p.ents = compact ? ctx->ents.as<uint32_t>() : nullptr;
    p.umeta = compact ? ctx->umeta.as<uint4>() : nullptr;
    p.eoff = compact ? ctx->eoff.as<uint32_t>() : nullptr;
    p.total_dus = S.du;
    p.out = ctx->out.as<uint8_t>();
    p.counters = ctx->counters.as<uint32_t>();
    p.k0_flag = ctx->k0_flag.as<uint32_t>();
    p.k0_agg = ctx->k0_agg.as<uint64_t>();
    p.k2_flag = ctx->k2_flag.as<uint32_t>();
    p.k2_agg = ctx->k2_agg.as<uint64_t>();
    p.stats = ctx->stats.as<unsigned long long>();
    return PJG_OK;
}

// blob_lo/blob_hi: the one caller allocation every file lies in (the blob
// API), or null — then the scans are copied from the caller's buffers only
// (packed into the pinned stage), except for a single file, whose scan is
// one range of that file.
int batch_create_impl(pjg_ctx* ctx, size_t n, const uint8_t* const* files, const size_t* sizes,
                      const pjg_config* cfg, const uint8_t* blob_lo, const uint8_t* blob_hi, pjg_batch** out) {
    *out = nullptr;
    int st = 0;
    if (!validate_cfg(ctx, cfg, &st)) return st;
    if (ctx->busy) return fail(ctx, PJG_INVALID_ARGUMENT, "one live batch per context");
    CU(cudaSetDevice(ctx->device), "cudaSetDevice");
    auto b = std::make_unique<pjg_batch>();
    b->ctx = ctx;
    b->cfg = *cfg;
    b->n = n;
    // PJG_HOST_TIMING=1: per-phase planning times on stderr (diagnostics)
    static const bool timing = getenv("PJG_HOST_TIMING") != nullptr;
    auto t_last = std::chrono::steady_clock::now();
    auto mark = [&](const char* what) {
        if (!timing) return;
        auto t = std::chrono::steady_clock::now();
        fprintf(stderr, "pjg_batch_create %-10s %8.3f ms\n", what,
                std::chrono::duration<double, std::milli>(t - t_last).count());
        t_last = t;
    };
    b->swap_pool(ctx->pool);
    b->dev_state.clear();
    b->host_status.resize(n);
    b->info.resize(n);
    // descriptors are written straight into their pinned upload buffer
    CU(ctx->desc_host.ensure(n * sizeof(ImgDesc) + 16), "cudaMallocHost(desc)");
    ImgDesc* const desc = static_cast<ImgDesc*>(ctx->desc_host.p);
    b->desc = desc;
    mark("arrays");

    // ---- phase A (parallel, contiguous image chunks): header parse, geometry,
    // per-image descriptor fields, table dedup against a per-worker unique list
    struct Worker {
        std::vector<HuffSpec> huff;  // unique specs, first-occurrence order
        std::vector<uint8_t> huff_dc;
        std::vector<std::array<uint16_t, 64>> quant;
        const uint8_t* lo = nullptr;
        const uint8_t* hi = nullptr;
        uint64_t raw_sum = 0, n_ok = 0, n_dri = 0;
    };
    auto same_spec = [](const HuffSpec& a, const HuffSpec& c) {
        return a.counts == c.counts && a.symbols.size() == c.symbols.size() &&
               std::memcmp(a.symbols.data(), c.symbols.data(), a.symbols.size()) == 0;
    };
    const bool allow_dri = cfg->restart_intervals != 0;
    const uint64_t sb = cfg->subsequence_bits;
    const unsigned hw = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
    const unsigned nw = (n >= 1024 && hw > 1) ? hw : 1;
    const size_t chunk = (n + nw - 1) / nw;
    std::vector<Worker> wk(nw);
    auto phase_a = [&](unsigned w) {
        Worker& W = wk[w];
        auto local_huff = [&](const HuffSpec& s, bool dc) -> uint16_t {
            for (size_t u = 0; u < W.huff.size(); ++u)
                if (W.huff_dc[u] == dc && same_spec(W.huff[u], s)) return uint16_t(u);
            W.huff.push_back(s);
            W.huff_dc.push_back(dc);
            return uint16_t(W.huff.size() - 1);
        };
        auto local_quant = [&](const std::array<uint16_t, 64>& q) -> uint16_t {
            for (size_t u = 0; u < W.quant.size(); ++u)
                if (std::memcmp(W.quant[u].data(), q.data(), 128) == 0) return uint16_t(u);
            W.quant.push_back(q);
            return uint16_t(W.quant.size() - 1);
        };
        const size_t i1 = std::min(n, (w + 1) * chunk);
        for (size_t i = w * chunk; i < i1; ++i) {
            Header h = parse_header(files[i], sizes[i], allow_dri);
            fill_info(h, cfg->output, sizes[i], &b->info[i]);
            ImgDesc& d = desc[i];
            std::memset(&d, 0, sizeof(d));
            d.out_mode = cfg->output;
            d.n_int = 1;
            // extract_scan of nothing → unstuff throws EmptyScan
            if (h.status == kOk && sizes[i] == h.scan_start) h.status = kEmptyScan;
            b->host_status[i] = h.status;
            if (h.status != kOk) continue;
            const size_t rl = sizes[i] - h.scan_start;
            const uint8_t* s = files[i] + h.scan_start;
            if (!W.lo || s < W.lo) W.lo = s;
            if (!W.hi || s + rl > W.hi) W.hi = s + rl;
            W.raw_sum += rl;
            ++W.n_ok;
            d.raw_off = uint64_t(reinterpret_cast<uintptr_t>(s));  // absolute until phase B
            d.raw_len = rl;
            d.deferred = h.table_status;
            d.width = h.width;
            d.height = h.height;
            d.mcus_x = h.mcus_x;
            d.mcus_y = h.mcus_y;
            d.ncomp = uint32_t(h.comps.size());
            d.dpm = h.dpm;
            d.h_max = h.h_max;
            d.v_max = h.v_max;
            uint32_t seen[4] = {0, 0, 0, 0};
            for (uint32_t k = 0; k < h.dpm; ++k) {
                uint32_t c = h.du_seq[k];
                d.du_comp |= uint64_t(c) << (4 * k);
                d.du_kslot |= uint64_t(seen[c]++) << (4 * k);
            }
            for (size_t c = 0; c < h.comps.size(); ++c) {
                d.comp_h[c] = h.comps[c].h;
                d.comp_v[c] = h.comps[c].v;
                d.plane_w[c] = h.comp_width(c);
                d.plane_h[c] = h.comp_height(c);
                if (h.table_status == kOk) {
                    d.dc_tab[c] = local_huff(h.dc[h.comps[c].td], true);
                    d.ac_tab[c] = local_huff(h.ac[h.comps[c].ta], false);
                }
                d.q_tab[c] = local_quant(h.quant[h.comps[c].tq]);
            }
            if (h.table_status != kOk) continue;
            d.sub_count = (uint64_t(rl) * 8 + sb - 1) / sb;
            if (h.restart_interval && h.intervals() > 1) {
                ++W.n_dri;
                d.n_int = uint32_t(h.intervals());  // checked and finished in phase B
                d.ri = h.restart_interval;
            }
            d.expected = h.total_dus() * 64;
            d.mcus_per_tile = uint16_t(k4_mcus_per_tile(h.h_max, h.dpm));  // K4 warp tiles (<= 24 data units)
            d.tiles_x = (h.mcus_x + d.mcus_per_tile - 1) / d.mcus_per_tile;
        }
    };
    ctx->pool_threads.run(nw, phase_a);
    mark("parse");

    // ---- tables: merge the workers' unique lists (batches almost always share
    // a handful, so a linear memcmp scan over the unique ones beats any map)
    std::vector<DevHuff> huffs;
    std::vector<std::array<uint16_t, 64>> quants;
    std::vector<std::pair<const HuffSpec*, bool>> huff_src;  // unique specs (first occurrence)
    std::vector<const std::array<uint16_t, 64>*> quant_src;
    std::vector<float> wqs;  // per quant table: 64 K3 metadata weights (zig-zag order)
    static const uint8_t kZz2R[64] = {0,  1,  8,  16, 9,  2,  3,  10, 17, 24, 32, 25, 18, 11, 4,  5,
                                      12, 19, 26, 33, 40, 48, 41, 34, 27, 20, 13, 6,  7,  14, 21, 28,
                                      35, 42, 49, 56, 57, 50, 43, 36, 29, 22, 15, 23, 30, 37, 44, 51,
                                      58, 59, 52, 45, 38, 31, 39, 46, 53, 60, 61, 54, 47, 55, 62, 63};
    std::vector<std::vector<uint16_t>> huff_map(nw), quant_map(nw);
    for (unsigned w = 0; w < nw; ++w) {
        const Worker& W = wk[w];
        for (size_t u = 0; u < W.huff.size(); ++u) {
            const HuffSpec& s = W.huff[u];
            const bool dc = W.huff_dc[u] != 0;
            size_t g = 0;
            while (g < huff_src.size() && !(huff_src[g].second == dc && same_spec(*huff_src[g].first, s))) ++g;
            if (g == huff_src.size()) {
                DevHuff d;
                build_dev_huff(s, &d);
                build_fast(&d, dc);
                huffs.push_back(d);
                huff_src.emplace_back(&s, dc);
            }
            huff_map[w].push_back(uint16_t(g));
        }
        for (const auto& q : W.quant) {
            size_t g = 0;
            while (g < quant_src.size() && std::memcmp(quant_src[g]->data(), q.data(), 128) != 0) ++g;
            if (g == quant_src.size()) {
                std::array<uint16_t, 64> r{};
                // column-major (index v*8 + u for raster u*8 + v), the coefficient buffer's order
                for (int z = 0; z < 64; ++z) r[(kZz2R[z] & 7) * 8 + (kZz2R[z] >> 3)] = q[z];
                quants.push_back(r);
                quant_src.push_back(&q);
                // K3 metadata weights: w_u w_v Q per zig-zag position, w_u >= max_x |basis[u][x]|
                static const double kW[8] = {0.35356, 0.4904, 0.46195, 0.4904, 0.35356, 0.4904, 0.46195, 0.4904};
                for (int z = 0; z < 64; ++z)
                    wqs.push_back(float(kW[kZz2R[z] >> 3] * kW[kZz2R[z] & 7] * double(q[z]) * (1.0 + 1e-6)));
            }
            quant_map[w].push_back(uint16_t(g));
        }
    }

    // ---- phase B (serial prefix sums): raw placement, global table ids, layout
    const uint8_t* lo = nullptr;
    const uint8_t* hi = nullptr;
    uint64_t raw_sum = 0, n_ok = 0, n_dri = 0;
    for (const Worker& W : wk) {
        if (W.lo && (!lo || W.lo < lo)) lo = W.lo;
        if (W.hi && (!hi || W.hi > hi)) hi = W.hi;
        raw_sum += W.raw_sum;
        n_ok += W.n_ok;
        n_dri += W.n_dri;
    }
    // Internal subsequence size: a batch too small to give half the SMs a K1
    // CTA is decoded at sb / 2^k (>= 256 bits, a multiple of 32 dividing sb) — more
    // threads for a latency-bound decode.  The decomposition is unique, so the
    // results do not change; every boundary at the configured sb is also one at
    // the internal size, and the sync-state dump aggregates back to the
    // configured partition.  Restart-interval batches keep sb (their
    // per-interval partitions are dumped as is).  PJG_SB_AUTO=0 turns it off.
    const uint64_t sb_int = internal_sb(sb, raw_sum * 8, n_dri == 0);
    b->sb_int = sb_int;
    // K0 tile size: 32 KB windows when the scans are large on average, else 8 KB
    uint32_t k0_bpt = (n_ok && raw_sum / n_ok >= 48 * 1024) ? kK0BigBpt : kK0SmallBpt;
    if (const char* e = getenv("PJG_K0_BPT"))  // override (A/B experiments): 16 or 64
        k0_bpt = atoi(e) == int(kK0BigBpt) ? kK0BigBpt : kK0SmallBpt;
    const uint64_t k0_tile = uint64_t(kK0Threads) * k0_bpt;
    // raw extent: one copy of the caller's region [lo, hi) when it lies in
    // memory the caller owns (a single file, or a declared blob) and is not
    // much larger than the scans; otherwise pack the scans into the stage
    const bool owned = n_ok <= 1 || (blob_lo && lo >= blob_lo && hi <= blob_hi);
    b->packed = !(lo && owned && uint64_t(hi - lo) <= raw_sum + raw_sum / 2 + (1u << 20));
    // Per image: global table ids, the restart-interval check, and its counts
    // (K0 tiles, subsequences, data units, K4 tiles, output bytes, segments,
    // packed bytes) — pass 1, per worker chunk; chunk totals are scanned
    // serially; pass 2 assigns every image its offsets (and copies its scan
    // into the pinned stage when packing).
    struct Counts {
        uint64_t pack = 0, sub = 0, du = 0, outb = 0, seg = 0;
        uint32_t k0t = 0, k4t = 0, ndri = 0;
    };
    std::vector<Counts> ctot(nw + 1);
    std::vector<uint32_t> k0_first(n + 1), tile_first(n + 1);
    std::vector<uint64_t> sub_first(n + 1);
    auto pass1 = [&](unsigned w) {
        Counts t;
        const size_t i1 = std::min(n, (w + 1) * chunk);
        for (size_t i = w * chunk; i < i1; ++i) {
            ImgDesc& d = desc[i];
            if (b->host_status[i] != kOk) continue;
            const size_t rl = d.raw_len;
            const uint8_t* s = reinterpret_cast<const uint8_t*>(uintptr_t(d.raw_off));
            if (!b->packed) d.raw_off = uint64_t(s - lo);  // packed: assigned in pass 2 (16-aligned)
            for (uint32_t c = 0; c < d.ncomp; ++c) {
                if (d.deferred == kOk) {
                    d.dc_tab[c] = huff_map[w][d.dc_tab[c]];
                    d.ac_tab[c] = huff_map[w][d.ac_tab[c]];
                }
                d.q_tab[c] = quant_map[w][d.q_tab[c]];
            }
            if (b->packed) t.pack += align_up(rl, 16);
            // K0 tiles always run (scan checks precede table errors); 16-byte-grid windows
            t.k0t += uint32_t((((b->packed ? 0 : d.raw_off) & 15) + rl + k0_tile - 1) / k0_tile);
            if (d.deferred != kOk) continue;
            if (sb_int != sb) d.sub_count = (uint64_t(rl) * 8 + sb_int - 1) / sb_int;
            if (d.n_int > 1) {
                // restart intervals: one subsequence partition per interval (K0b), at
                // most ceil(bits / sb) + intervals subsequences; segment bit offsets
                // are 32-bit
                if (uint64_t(rl) * 8 >= (1ull << 32)) {
                    b->host_status[i] = kUnsupportedFeature;
                    d.n_int = 1;
                    d.ri = 0;
                    d.expected = 0;
                    d.mcus_per_tile = 0;
                    d.tiles_x = 0;
                    d.pad1 = 1;  // placed in pass 2 like an accepted scan (K0 still runs)
                    continue;
                }
                t.seg += d.n_int + 1;
                d.sub_count += d.n_int;
                ++t.ndri;
            }
            t.sub += d.sub_count;
            t.du += d.expected / 64;
            t.k4t += d.tiles_x * d.mcus_y;
            t.outb += align_up(b->info[i].output_bytes, 256);
        }
        ctot[w] = t;
    };
    auto run_chunks = [&](const std::function<void(unsigned)>& fn) { ctx->pool_threads.run(nw, fn); };
    run_chunks(pass1);
    // exclusive scan of the chunk totals
    Counts run;
    for (unsigned w = 0; w <= nw; ++w) {
        const Counts t = w < nw ? ctot[w] : Counts{};
        ctot[w] = run;
        run.pack += t.pack;
        run.sub += t.sub;
        run.du += t.du;
        run.outb += t.outb;
        run.seg += t.seg;
        run.k0t += t.k0t;
        run.k4t += t.k4t;
        run.ndri += t.ndri;
    }
    const uint64_t pack_off = run.pack, sub = run.sub, du = run.du, outb = run.outb, seg_total = run.seg;
    const uint32_t k0t = run.k0t, k4t = run.k4t;
    std::vector<uint32_t> dri(run.ndri);  // images with restart intervals
    if (b->packed) CU(ctx->stage.ensure(pack_off + 64), "cudaMallocHost(stage)");
    uint8_t* const stage = b->packed ? static_cast<uint8_t*>(ctx->stage.p) : nullptr;
    std::vector<const uint8_t*> srcp(b->packed ? n : 0, nullptr);  // packed: each scan's source
    auto pass2 = [&](unsigned w) {
        Counts t = ctot[w];
        const size_t i1 = std::min(n, (w + 1) * chunk);
        for (size_t i = w * chunk; i < i1; ++i) {
            ImgDesc& d = desc[i];
            k0_first[i] = t.k0t;
            tile_first[i] = t.k4t;
            sub_first[i] = t.sub;
            d.sub_first = t.sub;
            d.du_first = t.du;
            d.out_off = t.outb;
            if (b->host_status[i] != kOk) {
                if (d.pad1) {  // a restart-interval scan rejected in pass 1 still runs K0
                    d.pad1 = 0;
                    const size_t rl = d.raw_len;
                    if (b->packed) {
                        srcp[i] = reinterpret_cast<const uint8_t*>(uintptr_t(d.raw_off));
                        d.raw_off = t.pack;
                        t.pack += align_up(rl, 16);
                    }
                    t.k0t += uint32_t(((d.raw_off & 15) + rl + k0_tile - 1) / k0_tile);
                }
                continue;
            }
            const size_t rl = d.raw_len;
            if (b->packed) {
                srcp[i] = reinterpret_cast<const uint8_t*>(uintptr_t(d.raw_off));
                d.raw_off = t.pack;
                t.pack += align_up(rl, 16);
            }
            t.k0t += uint32_t(((d.raw_off & 15) + rl + k0_tile - 1) / k0_tile);
            if (d.deferred != kOk) continue;
            if (d.n_int > 1) {
                d.seg_first = t.seg;
                t.seg += d.n_int + 1;
                dri[t.ndri++] = uint32_t(i);
            }
            t.sub += d.sub_count;
            t.du += d.expected / 64;
            t.k4t += d.tiles_x * d.mcus_y;
            t.outb += align_up(b->info[i].output_bytes, 256);
        }
    };
    run_chunks(pass2);
    if (b->packed) {  // the scans into the pinned stage, images interleaved across workers
        auto copy = [&](unsigned w) {
            for (size_t i = w; i < n; i += nw)
                if (srcp[i]) std::memcpy(stage + desc[i].raw_off, srcp[i], desc[i].raw_len);
        };
        run_chunks(copy);
    }
    k0_first[n] = k0t;
    tile_first[n] = k4t;
    sub_first[n] = sub;
    if (huffs.empty()) huffs.emplace_back();  // keep pointers valid
    if (quants.empty()) quants.emplace_back();
    b->n_huff = uint32_t(huffs.size());
    b->n_quant = uint32_t(quants.size());
    b->k0_tiles = k0t;
    b->k4_tiles = k4t;
    b->total_subs = sub;
    b->total_dus = du;
    b->seg_total = seg_total;
    b->out_bytes = outb;
    b->k1_ctas = uint32_t((sub + kK1Own - 1) / kK1Own);
    b->k2_tiles = uint32_t((sub + kK2Threads - 1) / kK2Threads);
    mark("layout");

    // ---- raw bytes: user region or the pinned stage (filled in pass 2)
    if (b->packed) {
        b->raw_src = stage;
        b->raw_bytes = pack_off;
    } else {
        b->raw_src = lo;
        b->raw_bytes = lo ? uint64_t(hi - lo) : 0;
    }

    mark("raw");
    if (timing)
        fprintf(stderr, "pjg_batch_create packed=%d raw_bytes=%llu pinned=%d\n", int(b->packed),
                (unsigned long long)b->raw_bytes, int(b->raw_src == ctx->stage.p));
    // ---- meta blob
    size_t o = 0;
    b->m_desc = o;
    o = align_up(o + n * sizeof(ImgDesc), 16);
    b->m_state = o;
    o = align_up(o + n * sizeof(ImgState), 16);
    b->m_huff = o;
    o = align_up(o + huffs.size() * sizeof(DevHuff), 16);
    b->m_quant = o;
    o = align_up(o + quants.size() * 128, 16);
    b->m_wq = o;
    o = align_up(o + quants.size() * 64 * sizeof(float), 16);
    b->m_basis = o;
    o = align_up(o + 64 * sizeof(double), 16);
    b->m_k0 = o;
    o = align_up(o + (n + 1) * 4, 16);
    b->m_tile = o;
    o = align_up(o + (n + 1) * 4, 16);
    b->m_sub = o;
    o = align_up(o + (n + 1) * 8, 16);
    // image lookup tables: K0 tile -> image, subsequence (c << kSubImgShift) -> image
    const uint64_t n_subimg = ((sub + (1u << kSubImgShift) - 1) >> kSubImgShift) + 2;
    b->m_k0img = o;
    o = align_up(o + (uint64_t(k0t) + 1) * 4, 16);
    b->m_subimg = o;
    o = align_up(o + n_subimg * 4, 16);
    b->m_dri = o;
    o = align_up(o + (dri.size() + 1) * 4, 16);
    b->m_total = o;
    CU(ctx->meta_host.ensure(o), "cudaMallocHost(meta)");
    uint8_t* mh = static_cast<uint8_t*>(ctx->meta_host.p);
    // [m_desc, m_state) of the device blob comes from ctx->desc_host (see upload)
    for (size_t i = 0; i < n; ++i) {
        ImgState s{};
        s.status = b->host_status[i];
        std::memcpy(mh + b->m_state + i * sizeof(ImgState), &s, sizeof(s));
    }
    std::memcpy(mh + b->m_huff, huffs.data(), huffs.size() * sizeof(DevHuff));
    std::memcpy(mh + b->m_quant, quants.data(), quants.size() * 128);
    if (!wqs.empty()) std::memcpy(mh + b->m_wq, wqs.data(), wqs.size() * sizeof(float));
    std::memcpy(mh + b->m_basis, ctx->basis, 64 * sizeof(double));
    std::memcpy(mh + b->m_k0, k0_first.data(), (n + 1) * 4);
    std::memcpy(mh + b->m_tile, tile_first.data(), (n + 1) * 4);
    std::memcpy(mh + b->m_sub, sub_first.data(), (n + 1) * 8);
    if (!dri.empty()) std::memcpy(mh + b->m_dri, dri.data(), dri.size() * 4);
    {
        uint32_t* k0img = reinterpret_cast<uint32_t*>(mh + b->m_k0img);
        for (size_t i = 0; i < n; ++i)
            for (uint32_t t = k0_first[i]; t < k0_first[i + 1]; ++t) k0img[t] = uint32_t(i);
        uint32_t* subimg = reinterpret_cast<uint32_t*>(mh + b->m_subimg);
        size_t k = 0;
        for (uint64_t c = 0; c < n_subimg; ++c) {
            const uint64_t g = c << kSubImgShift;
            // largest k < n with sub_first[k] <= g (find_seg semantics)
            while (k + 1 < n && sub_first[k + 1] <= g) ++k;
            subimg[c] = uint32_t(k);
        }
    }

    mark("meta");
    CU(ctx->meta.ensure(o), "cudaMalloc(meta)");
    {
        PlanSummary S;
        S.n = n;
        S.sub = sub;
        S.du = du;
        S.outb = outb;
        S.seg_total = seg_total;
        S.k0t = k0t;
        S.k4t = k4t;
        S.ndri = uint32_t(dri.size());
        S.n_huff = uint32_t(huffs.size());
        S.n_quant = uint32_t(quants.size());
        S.k0_bpt = k0_bpt;
        S.sb = sb;
        S.sb_int = sb_int;
        S.n_ok = n_ok;
        S.bits = 0;
        for (size_t i = 0; i < n; ++i)
            if (b->host_status[i] == kOk) {
                S.bits += desc[i].raw_len * 8;
                S.max_du = std::max<uint64_t>(S.max_du, desc[i].expected / 64);
            }
        S.all420 = cfg->output == PJG_OUT_RGB && n_ok > 0;
        for (size_t i = 0; i < n && S.all420; ++i)
            if (b->host_status[i] == kOk)
                S.all420 = desc[i].ncomp == 3 && desc[i].h_max == 2 && desc[i].v_max == 2;
        uint8_t* md = ctx->meta.as<uint8_t>();
        MetaPtrs M{md + b->m_desc, md + b->m_state, md + b->m_huff, md + b->m_quant, md + b->m_wq,
                   md + b->m_basis, md + b->m_k0, md + b->m_tile, md + b->m_sub, md + b->m_k0img,
                   md + b->m_subimg, md + b->m_dri};
        if ((st = finish_plan(ctx, b.get(), S, M))) return st;
    }
    mark("reserve");

    ctx->busy = true;
    *out = b.release();
    return PJG_OK;
}

}  // namespace

int pjg_batch_create(pjg_ctx* ctx, size_t n, const uint8_t* const* files, const size_t* sizes,
                     const pjg_config* cfg, pjg_batch** out) {
    if (!ctx || !out || (n && (!files || !sizes))) return PJG_INVALID_ARGUMENT;
    return batch_create_impl(ctx, n, files, sizes, cfg, nullptr, nullptr, out);
}

int pjg_batch_create_blob(pjg_ctx* ctx, const uint8_t* blob, size_t blob_bytes, size_t n, const uint64_t* offsets,
                          const size_t* sizes, const pjg_config* cfg, pjg_batch** out) {
    if (!ctx || !out || (n && (!blob || !offsets || !sizes))) return PJG_INVALID_ARGUMENT;
    std::vector<const uint8_t*> files(n);
    for (size_t i = 0; i < n; ++i) {
        if (offsets[i] > blob_bytes || sizes[i] > blob_bytes - offsets[i])
            return fail(ctx, PJG_INVALID_ARGUMENT, "file outside the blob");
        files[i] = blob + offsets[i];
    }
    return batch_create_impl(ctx, n, files.data(), sizes, cfg, blob, blob + blob_bytes, out);
}

// Device-side planning (devplan.cu): the files go up whole
// in one copy; the marker walk, table dedup/build and layout run as kernels;
// the host reads back one small totals record to size the decode.
int pjg_batch_create_device(pjg_ctx* ctx, const uint8_t* blob, size_t blob_bytes, size_t n,
                            const uint64_t* offsets, const size_t* sizes, const pjg_config* cfg, pjg_batch** out) {
    if (!ctx || !out || (n && (!blob || !offsets || !sizes))) return PJG_INVALID_ARGUMENT;
    *out = nullptr;
    int st = 0;
    if (!validate_cfg(ctx, cfg, &st)) return st;
    if (ctx->busy) return fail(ctx, PJG_INVALID_ARGUMENT, "one live batch per context");
    uint64_t tot = 0;
    for (size_t i = 0; i < n; ++i) {
        if (offsets[i] > blob_bytes || sizes[i] > blob_bytes - offsets[i])
            return fail(ctx, PJG_INVALID_ARGUMENT, "file outside the blob");
        tot += sizes[i];
    }
    CU(cudaSetDevice(ctx->device), "cudaSetDevice");
    cudaStream_t s = ctx->stream;
    auto b = std::make_unique<pjg_batch>();
    b->ctx = ctx;
    b->cfg = *cfg;
    b->n = n;
    b->devplan = true;
    b->swap_pool(ctx->pool);
    b->dev_state.clear();
    b->host_status.assign(n, 0);
    b->info.resize(n);
    // the host planner's heuristics on the files' bytes (scans are ~all of them)
    const uint64_t sb = cfg->subsequence_bits;
    const uint64_t sb_int = internal_sb(sb, tot * 8, !cfg->restart_intervals);
    uint32_t k0_bpt = (n && tot / n >= 48 * 1024) ? kK0BigBpt : kK0SmallBpt;
    if (const char* e = getenv("PJG_K0_BPT")) k0_bpt = atoi(e) == int(kK0BigBpt) ? kK0BigBpt : kK0SmallBpt;

    // ---- device layout: meta (desc, state, basis, prefix arrays, DRI list),
    // plan scratch (inputs, headers, dedup table, uniques, counts, totals)
    const size_t nn = std::max<size_t>(n, 1);
    size_t o = 0;
    b->m_desc = o;
    o = align_up(o + nn * sizeof(ImgDesc), 16);
    b->m_state = o;
    o = align_up(o + nn * sizeof(ImgState), 16);
    b->m_basis = o;
    o = align_up(o + 64 * sizeof(double), 16);
    b->m_k0 = o;
    o = align_up(o + (nn + 1) * 4, 16);
    b->m_tile = o;
    o = align_up(o + (nn + 1) * 4, 16);
    b->m_sub = o;
    o = align_up(o + (nn + 1) * 8, 16);
    b->m_dri = o;
    o = align_up(o + (nn + 1) * 4, 16);
    b->m_total = o;
    CU(ctx->meta.ensure(o), "cudaMalloc(meta)");
    const uint64_t refs = 9 * uint64_t(nn) + 16;
    uint64_t H = 64;
    while (H < 2 * refs) H <<= 1;
    const uint32_t nblk = uint32_t((nn + 255) / 256);
    size_t q = 0;
    const size_t p_off = q;  // offsets then sizes, contiguous: one upload of the pinned pair
    const size_t p_size = q + nn * 8;
    q = align_up(q + nn * 16, 16);
    const size_t p_hdr = q;
    q = align_up(q + nn * sizeof(DevHdr), 16);
    const size_t p_hkeys = q;
    q = align_up(q + H * 8, 16);
    const size_t p_hval = q;
    q = align_up(q + H * 4, 16);
    const size_t p_cnts = q;
    q = align_up(q + kPlanCounters * 4, 16);
    const size_t p_tot = q;
    q = align_up(q + sizeof(PlanTotals), 16);
    const size_t zero_end = q;  // [p_hkeys, zero_end) is zeroed per plan
    const size_t p_hrep = q;
    q = align_up(q + H * sizeof(TabRep), 16);
    const size_t p_uh = q;
    q = align_up(q + refs * sizeof(TabRep), 16);
    const size_t p_uq = q;
    q = align_up(q + refs * sizeof(TabRep), 16);
    const size_t p_state0 = q;
    q = align_up(q + nn * sizeof(ImgState), 16);
    const size_t p_info = q;
    q = align_up(q + nn * sizeof(pjg_image_info), 16);
    const size_t p_cnt = q;
    q = align_up(q + nn * sizeof(Cnt), 16);
    const size_t p_blk = q;
    q = align_up(q + (nblk + 1) * sizeof(Cnt), 16);
    CU(ctx->plan.ensure(q), "cudaMalloc(plan)");
    CU(ctx->raw.ensure(blob_bytes + 64), "cudaMalloc(raw)");
    CU(ctx->ubuf.ensure(blob_bytes + 64), "cudaMalloc(ubuf)");
    // pinned staging: offsets, sizes, basis; totals come back here
    const size_t h_tot = align_up(nn * 16 + 64 * sizeof(double), 16);
    CU(ctx->plan_host.ensure(h_tot + sizeof(PlanTotals)), "cudaMallocHost(plan)");
    uint8_t* ph = static_cast<uint8_t*>(ctx->plan_host.p);
    std::memcpy(ph, offsets, n * 8);
    for (size_t i = 0; i < n; ++i) reinterpret_cast<uint64_t*>(ph + nn * 8)[i] = sizes[i];
    std::memcpy(ph + nn * 16, ctx->basis, 64 * sizeof(double));

    uint8_t* pd = ctx->plan.as<uint8_t>();
    uint8_t* md = ctx->meta.as<uint8_t>();
    cudaPointerAttributes pa{};
    const bool dev_blob = cudaPointerGetAttributes(&pa, blob) == cudaSuccess && pa.type == cudaMemoryTypeDevice;
    cudaGetLastError();
    CU(cudaEventRecord(ctx->ev[0], s), "ev");
    if (blob_bytes)
        CU(cudaMemcpyAsync(ctx->raw.p, blob, blob_bytes, dev_blob ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, s),
           "H2D files");
    CU(cudaMemcpyAsync(pd + p_off, ph, nn * 16, cudaMemcpyHostToDevice, s), "H2D offsets");  // offsets, sizes
    CU(cudaMemcpyAsync(md + b->m_basis, ph + nn * 16, 64 * sizeof(double), cudaMemcpyHostToDevice, s), "H2D basis");
    CU(cudaEventRecord(ctx->ev[1], s), "ev");
    CU(cudaMemsetAsync(pd + p_hkeys, 0, zero_end - p_hkeys, s), "memset plan");

    PlanParams P{};
    P.raw = ctx->raw.as<uint8_t>();
    P.offsets = reinterpret_cast<const uint64_t*>(pd + p_off);
    P.sizes = reinterpret_cast<const uint64_t*>(pd + p_size);
    P.n = uint32_t(n);
    P.allow_dri = cfg->restart_intervals != 0;
    P.out_mode = cfg->output;
    P.k0_bpt = k0_bpt;
    P.sb_int = sb_int;
    P.hdr = reinterpret_cast<DevHdr*>(pd + p_hdr);
    P.hkeys = reinterpret_cast<uint64_t*>(pd + p_hkeys);
    P.hval = reinterpret_cast<uint32_t*>(pd + p_hval);
    P.hrep = reinterpret_cast<TabRep*>(pd + p_hrep);
    P.hmask = uint32_t(H - 1);
    P.counters = reinterpret_cast<uint32_t*>(pd + p_cnts);
    P.uh = reinterpret_cast<TabRep*>(pd + p_uh);
    P.uq = reinterpret_cast<TabRep*>(pd + p_uq);
    P.desc = reinterpret_cast<ImgDesc*>(md + b->m_desc);
    P.state = reinterpret_cast<ImgState*>(md + b->m_state);
    P.state0 = reinterpret_cast<ImgState*>(pd + p_state0);
    P.info = reinterpret_cast<pjg_image_info*>(pd + p_info);
    P.k0_first = reinterpret_cast<uint32_t*>(md + b->m_k0);
    P.tile_first = reinterpret_cast<uint32_t*>(md + b->m_tile);
    P.sub_first = reinterpret_cast<uint64_t*>(md + b->m_sub);
    P.dri = reinterpret_cast<uint32_t*>(md + b->m_dri);
    P.totals = reinterpret_cast<PlanTotals*>(pd + p_tot);
    P.cnt = reinterpret_cast<Cnt*>(pd + p_cnt);
    P.blk = reinterpret_cast<Cnt*>(pd + p_blk);
    if (n) {
        launch_plan_parse(P, s);
        CU(cudaGetLastError(), "plan launch");
    }
    PlanTotals T{};
    CU(cudaMemcpyAsync(ph + h_tot, pd + p_tot, sizeof(PlanTotals), cudaMemcpyDeviceToHost, s), "D2H totals");
    CU(cudaStreamSynchronize(s), "plan");
    std::memcpy(&T, ph + h_tot, sizeof(T));

    // ---- unique tables and lookup tables (sized by the totals)
    const uint32_t nh = std::max<uint32_t>(T.n_huff, 1), nq = std::max<uint32_t>(T.n_quant, 1);
    const uint64_t n_subimg = ((T.sub + (1u << kSubImgShift) - 1) >> kSubImgShift) + 2;
    size_t r = 0;
    b->m_huff = r;
    r = align_up(r + nh * sizeof(DevHuff), 16);
    b->m_quant = r;
    r = align_up(r + nq * 128, 16);
    b->m_wq = r;
    r = align_up(r + nq * 64 * sizeof(float), 16);
    b->m_k0img = r;
    r = align_up(r + (uint64_t(T.k0t) + 1) * 4, 16);
    b->m_subimg = r;
    r = align_up(r + n_subimg * 4, 16);
    CU(ctx->meta2.ensure(r), "cudaMalloc(meta2)");
    uint8_t* m2 = ctx->meta2.as<uint8_t>();
    TableOut TO{reinterpret_cast<DevHuff*>(m2 + b->m_huff), reinterpret_cast<uint16_t*>(m2 + b->m_quant),
                reinterpret_cast<float*>(m2 + b->m_wq), T.n_huff, T.n_quant};
    launch_plan_finish(P, TO, reinterpret_cast<uint32_t*>(m2 + b->m_k0img), reinterpret_cast<uint32_t*>(m2 + b->m_subimg),
                       n_subimg, s);
    CU(cudaGetLastError(), "plan launch");

    PlanSummary S;
    S.n = n;
    S.sub = T.sub;
    S.du = T.du;
    S.outb = T.outb;
    S.seg_total = T.seg;
    S.k0t = T.k0t;
    S.k4t = T.k4t;
    S.ndri = T.ndri;
    S.n_huff = nh;
    S.n_quant = nq;
    S.k0_bpt = k0_bpt;
    S.sb = sb;
    S.sb_int = sb_int;
    S.n_ok = T.n_ok;
    S.bits = T.bits;
    S.max_du = T.max_du;
    S.all420 = T.all420 != 0;
    MetaPtrs M{md + b->m_desc, md + b->m_state, m2 + b->m_huff, m2 + b->m_quant, m2 + b->m_wq,
               md + b->m_basis, md + b->m_k0, md + b->m_tile, md + b->m_sub, m2 + b->m_k0img,
               m2 + b->m_subimg, md + b->m_dri};
    b->raw_src = nullptr;
    b->raw_bytes = blob_bytes;
    b->packed = false;
    if ((st = finish_plan(ctx, b.get(), S, M))) return st;
    b->state0 = reinterpret_cast<const ImgState*>(pd + p_state0);
    b->dinfo = reinterpret_cast<const pjg_image_info*>(pd + p_info);
    b->uploaded = true;
    ctx->busy = true;
    *out = b.release();
    return PJG_OK;
}

namespace {
// Host copies of a device-planned batch's descriptors, header statuses and
// image infos (for the per-image API calls); a no-op for host-planned ones.
int host_view(const pjg_batch* cb) {
    pjg_batch* b = const_cast<pjg_batch*>(cb);
    if (!b->devplan || b->host_view) return PJG_OK;
    pjg_ctx* ctx = b->ctx;
    CU(cudaSetDevice(ctx->device), "cudaSetDevice");
    CU(ctx->desc_host.ensure(b->n * sizeof(ImgDesc) + 16), "cudaMallocHost(desc)");
    std::vector<ImgState> s0(b->n);
    if (b->n) {
        CU(cudaMemcpyAsync(ctx->desc_host.p, ctx->meta.as<uint8_t>() + b->m_desc, b->n * sizeof(ImgDesc),
                           cudaMemcpyDeviceToHost, ctx->stream),
           "D2H desc");
        CU(cudaMemcpyAsync(b->info.data(), b->dinfo, b->n * sizeof(pjg_image_info), cudaMemcpyDeviceToHost, ctx->stream),
           "D2H info");
        CU(cudaMemcpyAsync(s0.data(), b->state0, b->n * sizeof(ImgState), cudaMemcpyDeviceToHost, ctx->stream),
           "D2H status");
    }
    CU(cudaStreamSynchronize(ctx->stream), "host view");
    b->desc = static_cast<const ImgDesc*>(ctx->desc_host.p);
    for (size_t i = 0; i < b->n; ++i) b->host_status[i] = s0[i].status;
    b->host_view = true;
    return PJG_OK;
}
}  // namespace

int pjg_batch_upload(pjg_batch* b) {
    if (!b) return PJG_INVALID_ARGUMENT;
    if (b->devplan) return PJG_OK;  // the files went up with the plan
    pjg_ctx* ctx = b->ctx;
    CU(cudaSetDevice(ctx->device), "cudaSetDevice");
    CU(cudaEventRecord(ctx->ev[0], ctx->stream), "cudaEventRecord");
    if (b->raw_bytes)
        CU(cudaMemcpyAsync(ctx->raw.p, b->raw_src, b->raw_bytes, cudaMemcpyHostToDevice, ctx->stream),
           "H2D raw");
    if (b->m_state > b->m_desc)
        CU(cudaMemcpyAsync(ctx->meta.as<uint8_t>() + b->m_desc, ctx->desc_host.p, b->n * sizeof(ImgDesc),
                           cudaMemcpyHostToDevice, ctx->stream),
           "H2D desc");
    CU(cudaMemcpyAsync(ctx->meta.as<uint8_t>() + b->m_state, static_cast<uint8_t*>(ctx->meta_host.p) + b->m_state,
                       b->m_total - b->m_state, cudaMemcpyHostToDevice, ctx->stream),
       "H2D meta");
    CU(cudaEventRecord(ctx->ev[1], ctx->stream), "cudaEventRecord");
    b->uploaded = true;
    return PJG_OK;
}

namespace {
// The decode's stream work: status re-init, K0..K4, stage events, statuses and
// stats back.  Stage events are "external" records so that they also time a
// captured graph's replays.
int enqueue_decode(pjg_batch* b, cudaStream_t s) {
    pjg_ctx* ctx = b->ctx;
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    CU(cudaStreamIsCapturing(s, &cap), "capture status");
    const bool capturing = cap == cudaStreamCaptureStatusActive;
    auto ev = [&](int k) {
        return capturing ? cudaEventRecordWithFlags(ctx->ev[k], s, cudaEventRecordExternal) : cudaEventRecord(ctx->ev[k], s);
    };
    // status words are re-initialised so decode can be re-run on the same upload
    if (b->devplan) {
        if (b->n)
            CU(cudaMemcpyAsync(ctx->meta.as<uint8_t>() + b->m_state, b->state0, b->n * sizeof(ImgState),
                               cudaMemcpyDeviceToDevice, s),
               "D2D status");
    } else {
        uint8_t* mh = static_cast<uint8_t*>(ctx->meta_host.p);
        CU(cudaMemcpyAsync(ctx->meta.as<uint8_t>() + b->m_state, mh + b->m_state, b->n * sizeof(ImgState),
                           cudaMemcpyHostToDevice, s),
           "H2D status");
    }
    CU(cudaMemsetAsync(ctx->counters.p, 0, kNumCounters * 4, s), "memset counters");
    CU(cudaMemsetAsync(ctx->stats.p, 0, kNumStats * 8, s), "memset stats");
    CU(ev(2), "ev");
    if (b->prm.n_dri)  // interval starts not written by K0 stay ~0 (K0b flags them)
        CU(cudaMemsetAsync(ctx->segs.p, 0xFF, b->seg_total * sizeof(uint2), s), "memset segs");
    launch_k0_unstuff(b->prm, s);
    launch_k0b_segments(b->prm, s);
    CU(ev(3), "ev");
    launch_k1_sync(b->prm, s);
    launch_k1c_fixup(b->prm, s);
    CU(ev(4), "ev");
    launch_k2_scan(b->prm, s);
    CU(ev(5), "ev");
    if (b->total_dus) {
        if (b->prm.compact)
            CU(cudaMemsetAsync(ctx->umeta.p, 0, b->total_dus * 16, s), "memset umeta");
        else
            CU(cudaMemsetAsync(ctx->blkmeta.p, 0, b->total_dus * 8, s), "memset meta");
    }
    launch_k3_write(b->prm, s);
    // images whose entropy stage failed (or saw a run past a unit end): the
    // reference's exact semantics at the configured partition (K1x)
    launch_k1x_exact(b->prm, s);
    CU(ev(6), "ev");
    launch_k4_transform(b->prm, s);
    CU(cudaGetLastError(), "kernel launch");
    CU(ev(7), "ev");
    // statuses + stats back (small)
    uint8_t* sh = static_cast<uint8_t*>(ctx->status_host.p);
    CU(cudaMemcpyAsync(sh, ctx->meta.as<uint8_t>() + b->m_state, b->n * sizeof(ImgState),
                       cudaMemcpyDeviceToHost, s),
       "D2H status");
    CU(cudaMemcpyAsync(sh + align_up(b->n * sizeof(ImgState), 16), ctx->stats.p, kNumStats * 8,
                       cudaMemcpyDeviceToHost, s),
       "D2H stats");
    return PJG_OK;
}
}  // namespace

int pjg_batch_decode(pjg_batch* b) {
    if (!b) return PJG_INVALID_ARGUMENT;
    pjg_ctx* ctx = b->ctx;
    if (!b->uploaded) return fail(ctx, PJG_INVALID_ARGUMENT, "batch not uploaded");
    CU(cudaSetDevice(ctx->device), "cudaSetDevice");
    cudaStream_t s = ctx->stream;
    // Latency-bound batches (grids that do not fill the GPU) replay the whole
    // decode as one CUDA graph, captured at the first decode: one launch
    // instead of ~15 stream operations.  PJG_GRAPH=0/1 overrides.
    bool graph = b->k1_ctas < 2 * 148;
    if (const char* e = getenv("PJG_GRAPH")) graph = atoi(e) != 0;
    if (graph) {
        if (!b->gexec) {
            b->prm.epoch = ++ctx->epoch;  // fixed for the graph's replays (same inputs, same symbols)
            cudaGraph_t g = nullptr;
            CU(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal), "capture");
            const int st = enqueue_decode(b, s);
            const cudaError_t e = cudaStreamEndCapture(s, &g);
            if (st) {
                if (g) cudaGraphDestroy(g);
                return st;
            }
            CU(e, "capture");
            const cudaError_t ei = cudaGraphInstantiate(&b->gexec, g, 0);
            cudaGraphDestroy(g);
            CU(ei, "graph instantiate");
        }
        CU(cudaGraphLaunch(b->gexec, s), "graph launch");
    } else {
        b->prm.epoch = ++ctx->epoch;
        if (int st = enqueue_decode(b, s)) return st;
    }
    b->decoded = true;
    b->synced = false;
    return PJG_OK;
}

int pjg_batch_synchronize(pjg_batch* b, int32_t* statuses) {
    if (!b) return PJG_INVALID_ARGUMENT;
    pjg_ctx* ctx = b->ctx;
    if (!b->decoded) return fail(ctx, PJG_NOT_DECODED, "batch not decoded");
    CU(cudaSetDevice(ctx->device), "cudaSetDevice");
    CU(cudaStreamSynchronize(ctx->stream), "decode");
    if (!b->synced) {
        b->dev_state.resize(b->n);
        const uint8_t* sh = static_cast<const uint8_t*>(ctx->status_host.p);
        std::memcpy(b->dev_state.data(), sh, b->n * sizeof(ImgState));
        std::memcpy(b->stats, sh + align_up(b->n * sizeof(ImgState), 16), sizeof(b->stats));
        float ms = 0;
        cudaEventElapsedTime(&ms, ctx->ev[0], ctx->ev[1]);
        b->stage_ms[PJG_STAGE_UPLOAD] = ms;
        for (int k = 0; k < 5; ++k) {
            cudaEventElapsedTime(&ms, ctx->ev[2 + k], ctx->ev[3 + k]);
            b->stage_ms[PJG_STAGE_UNSTUFF + k] = ms;
        }
        b->synced = true;
    }
    if (statuses)
        for (size_t i = 0; i < b->n; ++i) statuses[i] = b->dev_state[i].status;
    return PJG_OK;
}

int pjg_batch_download(pjg_batch* b, uint8_t* const* outs, const size_t* caps) {
    if (!b || !outs) return PJG_INVALID_ARGUMENT;
    if (int hv = host_view(b)) return hv;
    pjg_ctx* ctx = b->ctx;
    int st = pjg_batch_synchronize(b, nullptr);
    if (st) return st;
    cudaEvent_t e0 = ctx->ev[0], e1 = ctx->ev[1];
    CU(cudaEventRecord(e0, ctx->stream), "ev");
    for (size_t i = 0; i < b->n; ++i) {
        if (!outs[i] || b->dev_state[i].status != 0) continue;
        uint64_t nb = b->info[i].output_bytes;
        if (caps && caps[i] < nb) return fail(ctx, PJG_CAPACITY, "output buffer too small");
        CU(cudaMemcpyAsync(outs[i], ctx->out.as<uint8_t>() + b->desc[i].out_off, nb, cudaMemcpyDeviceToHost,
                           ctx->stream),
           "D2H out");
    }
    CU(cudaEventRecord(e1, ctx->stream), "ev");
    CU(cudaStreamSynchronize(ctx->stream), "D2H");
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    b->stage_ms[PJG_STAGE_DOWNLOAD] = ms;
    return PJG_OK;
}

int pjg_batch_download_all(pjg_batch* b, void* host, size_t cap) {
    if (!b || !host) return PJG_INVALID_ARGUMENT;
    pjg_ctx* ctx = b->ctx;
    if (cap < b->out_bytes) return fail(ctx, PJG_CAPACITY, "output buffer too small");
    if (!b->decoded) return fail(ctx, PJG_NOT_DECODED, "batch not decoded");
    CU(cudaSetDevice(ctx->device), "cudaSetDevice");
    CU(cudaEventRecord(ctx->ev[0], ctx->stream), "ev");
    if (b->out_bytes)
        CU(cudaMemcpyAsync(host, ctx->out.p, b->out_bytes, cudaMemcpyDeviceToHost, ctx->stream), "D2H out");
    CU(cudaEventRecord(ctx->ev[1], ctx->stream), "ev");
    int st = pjg_batch_synchronize(b, nullptr);
    if (st) return st;
    float ms = 0;
    cudaEventElapsedTime(&ms, ctx->ev[0], ctx->ev[1]);
    b->stage_ms[PJG_STAGE_DOWNLOAD] = ms;
    return PJG_OK;
}

int pjg_batch_download_all_async(pjg_batch* b, void* host, size_t cap) {
    if (!b || !host) return PJG_INVALID_ARGUMENT;
    pjg_ctx* ctx = b->ctx;
    if (cap < b->out_bytes) return fail(ctx, PJG_CAPACITY, "output buffer too small");
    if (!b->decoded) return fail(ctx, PJG_NOT_DECODED, "batch not decoded");
    CU(cudaSetDevice(ctx->device), "cudaSetDevice");
    if (b->out_bytes)
        CU(cudaMemcpyAsync(host, ctx->out.p, b->out_bytes, cudaMemcpyDeviceToHost, ctx->stream), "D2H out");
    return PJG_OK;
}

uint64_t pjg_batch_output_offset(const pjg_batch* b, size_t i) {
    if (!b || i >= b->n) return 0;
    if (host_view(b)) return 0;
    return b->desc[i].out_off;
}

int pjg_batch_info(const pjg_batch* b, size_t i, pjg_image_info* info) {
    if (!b || i >= b->n || !info) return PJG_INVALID_ARGUMENT;
    if (int hv = host_view(b)) return hv;
    *info = b->info[i];
    return b->host_status[i];
}

const uint8_t* pjg_batch_device_output(const pjg_batch* b, size_t i) {
    if (!b || i >= b->n || host_view(b)) return nullptr;
    if (!b || i >= b->n || b->host_status[i] != 0 || b->desc[i].deferred != 0) return nullptr;
    return b->ctx->out.as<uint8_t>() + b->desc[i].out_off;
}

uint64_t pjg_batch_output_bytes(const pjg_batch* b) { return b ? b->out_bytes : 0; }

uint64_t pjg_batch_scan_bits(const pjg_batch* b) {
    if (!b || !b->synced) return 0;
    if (host_view(b)) return 0;
    uint64_t bits = 0;
    for (size_t i = 0; i < b->n; ++i)
        if (b->host_status[i] == 0 && i < b->dev_state.size() && b->dev_state[i].status == 0)
            bits += b->dev_state[i].bit_length;
    return bits;
}

uint32_t pjg_batch_kernel_launches(const pjg_batch* b) {
    if (!b) return 0;
    return kernel_launches(b->prm);
}

int pjg_batch_copy_outputs(pjg_batch* b, void* const* dst, const size_t* caps) {
    if (!b || !dst || !caps) return PJG_INVALID_ARGUMENT;
    if (int hv = host_view(b)) return hv;
    pjg_ctx* ctx = b->ctx;
    // only images that decoded: device failures (and deferred table errors,
    // which reserve no output) are known after the batch finished
    int st = pjg_batch_synchronize(b, nullptr);
    if (st) return st;
    for (size_t i = 0; i < b->n; ++i) {
        if (!dst[i]) continue;
        const uint64_t nb = b->info[i].output_bytes;
        if (caps[i] < nb) return fail(ctx, PJG_CAPACITY, "device output buffer too small");
        if (b->host_status[i] != 0 || b->dev_state[i].status != 0 || b->desc[i].deferred != 0 || nb == 0) continue;
        CU(cudaMemcpyAsync(dst[i], ctx->out.as<uint8_t>() + b->desc[i].out_off, nb, cudaMemcpyDeviceToDevice,
                           ctx->stream),
           "D2D output");
    }
    return PJG_OK;
}

int pjg_batch_stage_times(const pjg_batch* b, double* ms) {
    if (!b || !ms) return PJG_INVALID_ARGUMENT;
    for (int k = 0; k < PJG_NUM_STAGES; ++k) ms[k] = b->stage_ms[k];
    return PJG_OK;
}

int pjg_batch_sync_stats(const pjg_batch* b, uint64_t* stats) {
    if (!b || !stats) return PJG_INVALID_ARGUMENT;
    stats[0] = b->stats[kStatRoundsSum];
    stats[1] = b->stats[kStatRoundsMax];
    stats[2] = b->stats[kStatInterHops];
    stats[3] = b->stats[kStatFixPasses];
    stats[4] = b->stats[kStatReplays];
    stats[5] = b->stats[kStatAcUnits];
    stats[6] = b->stats[kStatEntries];
    stats[7] = b->prm.compact;
    return PJG_OK;
}

void pjg_batch_destroy(pjg_batch* b) {
    if (!b) return;
    if (b->ctx) {
        cudaSetDevice(b->ctx->device);
        cudaStreamSynchronize(b->ctx->stream);
        b->ctx->busy = false;
        b->swap_pool(b->ctx->pool);
    }
    if (b->gexec) cudaGraphExecDestroy(b->gexec);
    delete b;
}

int pjg_batch_dump_coefficients(const pjg_batch* b, size_t i, int pre_dc_zigzag, int16_t* out, size_t count) {
    if (!b || i >= b->n || !out) return PJG_INVALID_ARGUMENT;
    if (int hv = host_view(b)) return hv;
    pjg_ctx* ctx = b->ctx;
    const ImgDesc& d = b->desc[i];
    const uint64_t dus = uint64_t(d.mcus_x) * d.mcus_y * d.dpm;
    uint64_t nco = dus * 64;
    if (count < nco) return fail(ctx, PJG_CAPACITY, "coefficient buffer too small");
    if (b->host_status[i] != 0) return b->host_status[i];
    // compact batches keep no dense coefficients: expand the entries (debug tap)
    if (b->prm.compact) launch_k3d_densify(b->prm, ctx->stream);
    CU(cudaStreamSynchronize(ctx->stream), "sync");
    std::vector<int16_t> colmaj(nco), raster(nco);
    CU(cudaMemcpy(colmaj.data(), ctx->coef.as<int16_t>() + d.du_first * 64, nco * 2,
                  cudaMemcpyDeviceToHost),
       "D2H coef");
    // the device buffer holds each unit column-major (kernels.cu c_zz2c)
    for (uint64_t u = 0; u < nco; u += 64)
        for (int r = 0; r < 64; ++r) raster[u + r] = colmaj[u + (r & 7) * 8 + (r >> 3)];
    if (!pre_dc_zigzag) {
        std::memcpy(out, raster.data(), nco * 2);
        return PJG_OK;
    }
    static const uint8_t kZz2R[64] = {0,  1,  8,  16, 9,  2,  3,  10, 17, 24, 32, 25, 18, 11, 4,  5,
                                      12, 19, 26, 33, 40, 48, 41, 34, 27, 20, 13, 6,  7,  14, 21, 28,
                                      35, 42, 49, 56, 57, 50, 43, 36, 29, 22, 15, 23, 30, 37, 44, 51,
                                      58, 59, 52, 45, 38, 31, 39, 46, 53, 60, 61, 54, 47, 55, 62, 63};
    int32_t last[3] = {0, 0, 0};
    bool seen[3] = {false, false, false};
    for (uint64_t u = 0; u < dus; ++u) {
        const int16_t* r = raster.data() + u * 64;
        int16_t* z = out + u * 64;
        for (int k = 0; k < 64; ++k) z[k] = r[kZz2R[k]];
        unsigned comp = unsigned(d.du_comp >> (4 * (u % d.dpm))) & 15;
        int32_t abs_dc = z[0];
        // inverse of dc_prefix_sum (transform.hpp:56-74), exact mod 2^16
        if (seen[comp]) z[0] = int16_t(uint16_t(abs_dc - last[comp]));
        seen[comp] = true;
        last[comp] = abs_dc;
    }
    return PJG_OK;
}

int pjg_batch_dump_sync_states(const pjg_batch* b, size_t i, pjg_sync_entry* out, size_t cap, size_t* n_out) {
    if (!b || i >= b->n || !n_out) return PJG_INVALID_ARGUMENT;
    if (int hv = host_view(b)) return hv;
    pjg_ctx* ctx = b->ctx;
    int st = pjg_batch_synchronize(const_cast<pjg_batch*>(b), nullptr);
    if (st) return st;
    if (b->host_status[i] != 0) return b->host_status[i];
    const uint64_t L = b->dev_state[i].bit_length;
    // K1x-redone images hold the reference's entries at the configured partition
    const bool redone = (b->dev_state[i].exact & 2u) != 0;
    const uint64_t sbu = b->cfg.subsequence_bits, f = (b->sb_int && !redone) ? sbu / b->sb_int : 1;
    uint64_t N = (L + sbu - 1) / sbu;
    if (b->desc[i].n_int > 1) {  // restart intervals: the subsequences in use (K0b)
        uint2 last;
        CU(cudaMemcpy(&last, ctx->segs.as<uint2>() + b->desc[i].seg_first + b->desc[i].n_int, sizeof(uint2),
                      cudaMemcpyDeviceToHost),
           "D2H segs");
        N = last.y;
    }
    *n_out = N;
    if (!out) return PJG_OK;
    if (cap < N) return fail(ctx, PJG_CAPACITY, "sync state buffer too small");
    // internal subsequences (f per configured one when sb was split)
    const uint64_t Ni = (b->desc[i].n_int > 1 || redone) ? N : (L + b->sb_int - 1) / b->sb_int;
    std::vector<Entry> ents(Ni);
    std::vector<uint32_t> caps(Ni);
    const uint64_t g0 = b->desc[i].sub_first;
    if (Ni) {
        CU(cudaMemcpy(ents.data(), ctx->ent.as<Entry>() + g0, Ni * sizeof(Entry), cudaMemcpyDeviceToHost), "D2H ent");
        CU(cudaMemcpy(caps.data(), ctx->cap.as<uint32_t>() + g0, Ni * 4, cudaMemcpyDeviceToHost), "D2H cap");
        if (redone)
            for (uint64_t j = 0; j < Ni; ++j) caps[j] = ents[j].n;  // trimmed by K1x's offsets()
    }
    const uint64_t fk = b->desc[i].n_int > 1 ? 1 : f;
    for (uint64_t k = 0; k < N; ++k) {
        // the configured subsequence k = internal ones [k f, min((k+1) f, Ni)):
        // its entry is the last one's (same boundary), its slots their sum
        const uint64_t last = std::min((k + 1) * fk, Ni) - 1;
        uint64_t nn = 0;
        for (uint64_t j = k * fk; j <= last; ++j) nn += caps[j];
        out[k].p = ents[last].p;
        out[k].n = nn;
        out[k].c = czd_c(ents[last].czd);
        out[k].z = czd_z(ents[last].czd);
        out[k].divergent = czd_div(ents[last].czd) ? 1 : 0;
        out[k].pad = 0;
    }
    return PJG_OK;
}

int pjg_batch_dump_segment(const pjg_batch* b, size_t i, uint8_t* out, size_t cap, size_t* n_out) {
    if (!b || i >= b->n || !n_out) return PJG_INVALID_ARGUMENT;
    if (int hv = host_view(b)) return hv;
    pjg_ctx* ctx = b->ctx;
    int st = pjg_batch_synchronize(const_cast<pjg_batch*>(b), nullptr);
    if (st) return st;
    if (b->host_status[i] != 0) return b->host_status[i];
    const uint64_t bytes = b->dev_state[i].bit_length / 8;
    *n_out = bytes;
    if (!out) return PJG_OK;
    if (cap < bytes) return fail(ctx, PJG_CAPACITY, "segment buffer too small");
    if (bytes)
        CU(cudaMemcpy(out, ctx->ubuf.as<uint8_t>() + b->desc[i].raw_off, bytes, cudaMemcpyDeviceToHost),
           "D2H segment");
    return PJG_OK;
}

int pjg_decode_batch(pjg_ctx* ctx, size_t n, const uint8_t* const* files, const size_t* sizes,
                     const pjg_config* cfg, pjg_image_info* infos, uint8_t* const* outs,
                     const size_t* out_caps, int32_t* statuses) {
    if (!ctx) return PJG_INVALID_ARGUMENT;
    pjg_batch* b = nullptr;
    int st = pjg_batch_create(ctx, n, files, sizes, cfg, &b);
    if (st) return st;
    std::unique_ptr<pjg_batch, void (*)(pjg_batch*)> guard(b, pjg_batch_destroy);
    if ((st = pjg_batch_upload(b))) return st;
    if ((st = pjg_batch_decode(b))) return st;
    if ((st = pjg_batch_synchronize(b, statuses))) return st;
    if (infos)
        for (size_t i = 0; i < n; ++i) infos[i] = b->info[i];
    if (outs && (st = pjg_batch_download(b, outs, out_caps))) return st;
    return PJG_OK;
}

int pjg_decode(pjg_ctx* ctx, const uint8_t* file, size_t size, const pjg_config* cfg, pjg_image_info* info,
               uint8_t* out, size_t out_capacity) {
    int32_t status = 0;
    pjg_image_info tmp;
    uint8_t* outs[1] = {out};
    size_t caps[1] = {out_capacity};
    int st = pjg_decode_batch(ctx, 1, &file, &size, cfg, info ? info : &tmp, out ? outs : nullptr, caps, &status);
    if (st) return st;
    if (status) {
        if (ctx) ctx->err = pjg_status_name(status);
        return status;
    }
    return PJG_OK;
}

int pjg_upsample_and_convert(pjg_ctx* ctx, uint32_t width, uint32_t height, uint32_t nplanes,
                             const uint32_t* plane_w, const uint32_t* plane_h, const uint8_t* const* planes,
                             uint8_t* out_rgb) {
    if (!ctx || !plane_w || !plane_h || !planes || !out_rgb || nplanes < 1 || nplanes > 3)
        return PJG_INVALID_ARGUMENT;
    CU(cudaSetDevice(ctx->device), "cudaSetDevice");
    const uint64_t npx = uint64_t(width) * height;
    if (nplanes == 1) {  // grayscale passthrough (pipeline.hpp:171-176)
        for (uint32_t r = 0; r < height; ++r) std::memcpy(out_rgb + uint64_t(r) * width, planes[0] + uint64_t(r) * plane_w[0], width);
        return PJG_OK;
    }
    if (nplanes != 3) return fail(ctx, PJG_INVALID_ARGUMENT, "upsample_and_convert needs 1 or 3 planes");
    uint64_t sz[3], tot = 0;
    for (int c = 0; c < 3; ++c) {
        sz[c] = uint64_t(plane_w[c]) * plane_h[c];
        tot += align_up(sz[c], 256);
    }
    // the context's grow-only scratch (no allocation per call)
    CU(ctx->k5tmp.ensure(tot + npx * 3), "cudaMalloc(k5tmp)");
    uint8_t* d = ctx->k5tmp.as<uint8_t>();
    uint8_t* dp[3];
    uint64_t o = 0;
    for (int c = 0; c < 3; ++c) {
        dp[c] = d + o;
        CU(cudaMemcpyAsync(dp[c], planes[c], sz[c], cudaMemcpyHostToDevice, ctx->stream), "H2D planes");
        o += align_up(sz[c], 256);
    }
    launch_k5_color(dp[0], dp[1], dp[2], width, height, plane_w[0], plane_w[1], plane_h[1], plane_w[2], plane_h[2],
                    d + o, ctx->stream);
    CU(cudaGetLastError(), "k5 launch");
    CU(cudaMemcpyAsync(out_rgb, d + o, npx * 3, cudaMemcpyDeviceToHost, ctx->stream), "D2H rgb");
    CU(cudaStreamSynchronize(ctx->stream), "colour");
    return PJG_OK;
}

// The device planner's header parse (devparse.h) run on the host, for CPU
// tests: out = {status, table_status, width, height, ncomp, dpm, scan_start}.
int pjg_debug_device_parse(const uint8_t* file, size_t size, int allow_dri, int64_t* out) {
    if ((!file && size) || !out) return PJG_INVALID_ARGUMENT;
    // the file at an unaligned offset of a 16-byte-aligned buffer, as in a batch blob
    constexpr size_t kOff = 13;
    std::vector<uint4> buf(align_up(size + kOff, 16) / 16 + 2);
    std::memset(buf.data(), 0, buf.size() * 16);
    if (size) std::memcpy(reinterpret_cast<uint8_t*>(buf.data()) + kOff, file, size);
    DReader r;
    r.base = reinterpret_cast<const uint8_t*>(buf.data());
    r.f0 = kOff;
    r.size = size;
    DevHdr h;
    std::memset(&h, 0, sizeof(h));
    h.status = kMalformedHeader;
    h.h_max = h.v_max = 1;
    parse_file(r, allow_dri != 0, h);
    const int64_t v[7] = {h.status, h.table_status, h.width, h.height, h.ncomp, h.dpm, int64_t(h.scan_start)};
    std::memcpy(out, v, sizeof(v));
    return PJG_OK;
}

int pjg_debug_huff_decode(const uint8_t* counts16, const uint8_t* symbols, size_t nsym, const uint16_t* windows,
                          size_t nwin, uint32_t* out) {
    HuffSpec s;
    std::memcpy(s.counts.data(), counts16, 16);
    s.symbols.p = symbols;
    s.symbols.n = uint32_t(nsym);
    s.present = true;
    DevHuff d;
    int32_t st = build_dev_huff(s, &d);
    if (st) return -st;
    for (size_t i = 0; i < nwin; ++i) out[i] = huff_lookup(d, windows[i]);
    return 0;
}

int pjg_debug_fast_entry(const uint8_t* counts16, const uint8_t* symbols, size_t nsym, int dc,
                         const uint32_t* windows, size_t nwin, uint32_t* out) {
    HuffSpec s;
    std::memcpy(s.counts.data(), counts16, 16);
    s.symbols.p = symbols;
    s.symbols.n = uint32_t(nsym);
    s.present = true;
    DevHuff d;
    int32_t st = build_dev_huff(s, &d);
    if (st) return -st;
    build_fast(&d, dc != 0);
    for (size_t i = 0; i < nwin; ++i) {
        const uint32_t w = windows[i];
        uint32_t fe = d.fast[w >> (32 - kFastBits)];
        if ((fe & 0x3FFu) == kFastL2) fe = d.fast2[(fe >> 10) & 31u][(w >> (32 - kFastBits - 5)) & 31u];
        out[i] = fe;
    }
    return 0;
}

}  // extern "C"
