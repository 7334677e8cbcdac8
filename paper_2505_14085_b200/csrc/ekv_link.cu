// The emulated cloud -> edge link of the C ABI over NCCL (include/ekv_capi.h,
// "link"): the B200 counterpart of Sim::fetch_deep_layer -> submit_transfer
// (sim.cpp:802-814, 417-449), one process per GPU.  The cloud rank sends the
// compressed deep layers of its assembled context layer by layer
// (ncclSend, one NCCL group per layer, on the context's copy stream); the edge
// rank receives them straight into its context's storage and forwards the user
// rows layer-major on the compute stream, layer l's attention waiting only for
// layer l's receive (Eq. 20, cost_model.cpp:73-100, on real streams).
//
// NCCL is resolved at run time (dlopen of libnccl.so.2, reusing a copy already
// loaded into the process, e.g. PyTorch's), so libekv.so carries no link-time
// dependency and never mixes two NCCL builds in one process.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <string>
#include <vector>

#include "ekv_objects.h"

using namespace ekv;

namespace {

struct Nccl {
    ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
    ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
    ncclResult_t (*send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*group_start)() = nullptr;
    ncclResult_t (*group_end)() = nullptr;
    const char* (*error_string)(ncclResult_t) = nullptr;
};

const Nccl& nccl() {
    static Nccl n;
    static bool done = false;
    if (done) return n;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);  // the process's NCCL, if any
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
        const char* e = dlerror();
        throw Error(EKV_EUNSUPPORTED, std::string("link: libnccl.so.2 not found: ") + (e ? e : "?"));
    }
    auto sym = [&](const char* name) {
        void* p = dlsym(h, name);
        require(p != nullptr, std::string("link: NCCL symbol ") + name + " missing", EKV_EUNSUPPORTED);
        return p;
    };
    n.get_unique_id = (decltype(n.get_unique_id))sym("ncclGetUniqueId");
    n.comm_init_rank = (decltype(n.comm_init_rank))sym("ncclCommInitRank");
    n.comm_destroy = (decltype(n.comm_destroy))sym("ncclCommDestroy");
    n.send = (decltype(n.send))sym("ncclSend");
    n.recv = (decltype(n.recv))sym("ncclRecv");
    n.group_start = (decltype(n.group_start))sym("ncclGroupStart");
    n.group_end = (decltype(n.group_end))sym("ncclGroupEnd");
    n.error_string = (decltype(n.error_string))sym("ncclGetErrorString");
    done = true;
    return n;
}

void nccl_check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess)
        throw Error(EKV_ECUDA, std::string(what) + ": " + nccl().error_string(r));
}

// the four arrays of a context layer (bf16: K, V)
int layer_arrays(const ekv_kvctx_s* c, int l, void** p, size_t* n) {
    const ekv_model_s* m = c->model;
    const ekv_segment& sg = c->seg.at(l);
    const size_t rows = (size_t)m->cfg.num_heads * c->S, d = m->cfg.head_dim;
    const size_t cb = rows * d * sg.format / 8;
    p[0] = (void*)sg.k;
    p[1] = (void*)sg.v;
    n[0] = n[1] = cb;
    if (sg.format == EKV_KV_BF16) return 2;
    p[2] = (void*)sg.k_scales;
    p[3] = (void*)sg.v_scales;
    n[2] = n[3] = rows * (d / sg.group) * 4;
    return 4;
}

void check_layers(const ekv_kvctx_s* c, const int* layers, int n) {
    require(layers != nullptr || n == 0, "link: null layer list");
    for (int i = 0; i < n; ++i)
        require(layers[i] >= 0 && layers[i] < (int)c->seg.size(),
                "assemble_context: missing layer " + std::to_string(layers[i]));
}

}  // namespace

struct ekv_link_s {
    ekv_ctx_s* ctx = nullptr;
    ncclComm_t comm = nullptr;
    int rank = 0, nranks = 0;
};

extern "C" {

int ekv_link_unique_id(void* id_out) {
    return guard([&] {
        require(id_out != nullptr, "ekv_link_unique_id: null argument");
        ncclUniqueId id;
        nccl_check(nccl().get_unique_id(&id), "ncclGetUniqueId");
        std::memcpy(id_out, &id, sizeof(id));
    });
}

int ekv_link_create(ekv_ctx_t c, const void* id, int nranks, int rank, ekv_link_t* out) {
    return guard([&] {
        require(c && id && out, "ekv_link_create: null argument");
        require(nranks >= 1 && rank >= 0 && rank < nranks, "ekv_link_create: bad rank");
        set_dev(c);
        ncclUniqueId uid;
        std::memcpy(&uid, id, sizeof(uid));
        auto* l = new ekv_link_s();
        l->ctx = c;
        l->rank = rank;
        l->nranks = nranks;
        ncclResult_t r = nccl().comm_init_rank(&l->comm, nranks, uid, rank);
        if (r != ncclSuccess) {
            delete l;
            nccl_check(r, "ncclCommInitRank");
        }
        c->refs++;
        *out = l;
    });
}

int ekv_link_destroy(ekv_link_t l) {
    return guard([&] {
        if (!l) return;
        set_dev(l->ctx);
        cudaStreamSynchronize(l->ctx->copy);
        if (l->comm) nccl().comm_destroy(l->comm);
        ekv_ctx_s* c = l->ctx;
        delete l;
        release_ctx(c);
    });
}

int ekv_link_send_layers(ekv_link_t lk, ekv_kvctx_t src, const int* layers, int n, int peer,
                         float* seconds) {
    return guard([&] {
        require(lk && src, "ekv_link_send_layers: null argument");
        require(peer >= 0 && peer < lk->nranks && peer != lk->rank, "link: bad peer rank");
        check_layers(src, layers, n);
        ekv_ctx_s* c = lk->ctx;
        set_dev(c);
        cudaStream_t cp = c->copy;
        cudaEvent_t e0 = nullptr, e1 = nullptr, start = nullptr;
        EKV_CUDA(cudaEventCreate(&e0));
        EKV_CUDA(cudaEventCreate(&e1));
        EKV_CUDA(cudaEventCreateWithFlags(&start, cudaEventDisableTiming));
        // the layers are final once the context stream's queued work (e.g. build_deep_kv) is
        EKV_CUDA(cudaEventRecord(start, c->stream));
        EKV_CUDA(cudaStreamWaitEvent(cp, start, 0));
        EKV_CUDA(cudaEventRecord(e0, cp));
        for (int i = 0; i < n; ++i) {
            void* p[4];
            size_t nb[4];
            const int k = layer_arrays(src, layers[i], p, nb);
            nccl_check(nccl().group_start(), "ncclGroupStart");
            for (int a = 0; a < k; ++a) nccl_check(nccl().send(p[a], nb[a], ncclUint8, peer, lk->comm, cp), "ncclSend");
            nccl_check(nccl().group_end(), "ncclGroupEnd");
        }
        EKV_CUDA(cudaEventRecord(e1, cp));
        EKV_CUDA(cudaStreamSynchronize(cp));
        float ms = 0.f;
        EKV_CUDA(cudaEventElapsedTime(&ms, e0, e1));
        if (seconds) *seconds = ms * 1e-3f;
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        cudaEventDestroy(start);
    });
}

int ekv_link_recv_forward(ekv_link_t lk, ekv_session_t s, const int* layers, int n, int peer,
                          const float* emb_dev, int rows, float* out_dev, float* seconds) {
    return guard([&] {
        require(lk && s, "ekv_link_recv_forward: null argument");
        require(peer >= 0 && peer < lk->nranks && peer != lk->rank, "link: bad peer rank");
        ekv_kvctx_s* c = s->kv;
        check_layers(c, layers, n);
        ekv_ctx_s* ctx = lk->ctx;
        require(s->model->ctx == ctx, "link: the session lives on another context");
        if (rows > 0) {
            require(emb_dev != nullptr, "ekv_link_recv_forward: null embeddings");
            check_overflow(s, rows);
        }
        set_dev(ctx);
        cudaStream_t cp = ctx->copy;
        const int L = s->model->cfg.num_layers;
        std::vector<cudaEvent_t> ready(L, nullptr);
        cudaEvent_t e0 = nullptr, e1 = nullptr, start = nullptr;
        auto cleanup = [&] {
            for (auto& e : ready)
                if (e) cudaEventDestroy(e);
            for (cudaEvent_t e : {e0, e1, start})
                if (e) cudaEventDestroy(e);
        };
        try {
            EKV_CUDA(cudaEventCreate(&e0));
            EKV_CUDA(cudaEventCreate(&e1));
            EKV_CUDA(cudaEventCreateWithFlags(&start, cudaEventDisableTiming));
            EKV_CUDA(cudaEventRecord(start, ctx->stream));  // nothing reads the layers mid-receive
            EKV_CUDA(cudaStreamWaitEvent(cp, start, 0));
            EKV_CUDA(cudaEventRecord(e0, cp));
            for (int i = 0; i < n; ++i) {
                const int l = layers[i];
                void* p[4];
                size_t nb[4];
                const int k = layer_arrays(c, l, p, nb);
                nccl_check(nccl().group_start(), "ncclGroupStart");
                for (int a = 0; a < k; ++a)
                    nccl_check(nccl().recv(p[a], nb[a], ncclUint8, peer, lk->comm, cp), "ncclRecv");
                nccl_check(nccl().group_end(), "ncclGroupEnd");
                EKV_CUDA(cudaEventCreateWithFlags(&ready[l], cudaEventDisableTiming));
                EKV_CUDA(cudaEventRecord(ready[l], cp));
            }
            EKV_CUDA(cudaEventRecord(e1, cp));
            if (rows > 0) streamed_forward(s, emb_dev, rows, out_dev, ready.data(), nullptr, nullptr, nullptr);
            EKV_CUDA(cudaStreamSynchronize(cp));
            EKV_CUDA(cudaStreamSynchronize(ctx->stream));
            float ms = 0.f;
            EKV_CUDA(cudaEventElapsedTime(&ms, e0, e1));
            if (seconds) *seconds = ms * 1e-3f;
        } catch (...) {
            cudaStreamSynchronize(cp);
            cudaStreamSynchronize(ctx->stream);
            cleanup();
            throw;
        }
        cleanup();
    });
}

}  // extern "C"
