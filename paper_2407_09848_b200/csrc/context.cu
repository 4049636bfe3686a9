// Context, memory and error plumbing of libamgp.so.
#include <stdio.h>

#include "amgp_common.cuh"

static thread_local std::string g_last_error;
thread_local CaptureOverride amgp_capture;

void amgp_set_error(const std::string &msg) { g_last_error = msg; }

int amgp_fail(int code, const std::string &msg) {
    g_last_error = msg;
    return code;
}

int amgp_cuda_fail(cudaError_t e, const char *what, const char *file, int line) {
    char buf[512];
    snprintf(buf, sizeof(buf), "CUDA error %s (%s) in %s at %s:%d", cudaGetErrorName(e),
             cudaGetErrorString(e), what, file, line);
    g_last_error = buf;
    return e == cudaErrorMemoryAllocation ? AMGP_ENOMEM : AMGP_ECUDA;
}

extern "C" {

const char *amgp_last_error(void) { return g_last_error.c_str(); }

int amgp_version(void) { return 1; }

int amgp_ctx_create(int device, void *stream, amgp_ctx **out) {
    if (!out) return amgp_fail(AMGP_EINVAL, "amgp_ctx_create: out is NULL");
    int ndev = 0;
    AMGP_CUDA(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev)
        return amgp_fail(AMGP_EINVAL, "amgp_ctx_create: invalid device ordinal");
    AMGP_CUDA(cudaSetDevice(device));
    amgp_ctx *c = new amgp_ctx();
    c->device = device;
    if (stream) {
        c->stream = (cudaStream_t)stream;
    } else {
        cudaError_t e = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking);
        if (e != cudaSuccess) {
            delete c;
            return amgp_cuda_fail(e, "cudaStreamCreate", __FILE__, __LINE__);
        }
        c->own_stream = true;
    }
    cudaError_t e = cudaMalloc(&c->scalars, 64 * sizeof(double));
    if (e == cudaSuccess) e = cudaMallocHost(&c->host_scalars, 64 * sizeof(double));
    if (e == cudaSuccess) e = cudaMemset(c->scalars, 0, 64 * sizeof(double));
    if (e != cudaSuccess) {
        if (c->own_stream) cudaStreamDestroy(c->stream);
        cudaFree(c->scalars);
        delete c;
        return amgp_cuda_fail(e, "amgp_ctx_create alloc", __FILE__, __LINE__);
    }
    *out = c;
    return AMGP_OK;
}

int amgp_ctx_destroy(amgp_ctx *c) {
    if (!c) return AMGP_OK;
    cudaSetDevice(c->device);
    cudaStreamSynchronize(c->stream);
    ctx_free_comm(c);
    cudaFree(c->red_partial);
    cudaFree(c->scalars);
    cudaFreeHost(c->host_scalars);
    if (c->own_stream) cudaStreamDestroy(c->stream);
    if (c->io_h2d) cudaStreamDestroy(c->io_h2d);
    if (c->io_d2h) cudaStreamDestroy(c->io_d2h);
    delete c;
    return AMGP_OK;
}

int amgp_ctx_set_stream(amgp_ctx *c, void *stream) {
    if (!c) return amgp_fail(AMGP_EINVAL, "null context");
    std::lock_guard<std::mutex> g(c->mu);
    if (c->own_stream) {
        cudaStreamSynchronize(c->stream);
        cudaStreamDestroy(c->stream);
        c->own_stream = false;
    }
    if (stream) {
        c->stream = (cudaStream_t)stream;
    } else {
        AMGP_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
        c->own_stream = true;
    }
    return AMGP_OK;
}

int amgp_ctx_sync(amgp_ctx *c) {
    if (!c) return amgp_fail(AMGP_EINVAL, "null context");
    AMGP_CUDA(cudaStreamSynchronize(c->stream));
    return AMGP_OK;
}

int amgp_ctx_launch_count(amgp_ctx *c, int64_t *count) {
    if (!c || !count) return amgp_fail(AMGP_EINVAL, "null argument");
    *count = c->launches.load();
    return AMGP_OK;
}

int amgp_malloc(amgp_ctx *c, int64_t bytes, void **dptr) {
    if (!c || !dptr || bytes < 0) return amgp_fail(AMGP_EINVAL, "amgp_malloc: bad argument");
    AMGP_CUDA(cudaSetDevice(c->device));
    AMGP_CUDA(cudaMalloc(dptr, bytes > 0 ? (size_t)bytes : 8));
    return AMGP_OK;
}

int amgp_free(amgp_ctx *c, void *dptr) {
    if (!c) return amgp_fail(AMGP_EINVAL, "null context");
    if (dptr) {
        cudaStreamSynchronize(c->stream);
        AMGP_CUDA(cudaFree(dptr));
    }
    return AMGP_OK;
}

int amgp_memcpy_h2d(amgp_ctx *c, void *dst, const void *src, int64_t bytes) {
    if (!c) return amgp_fail(AMGP_EINVAL, "null context");
    if (bytes <= 0) return AMGP_OK;
    AMGP_CUDA(cudaMemcpyAsync(dst, src, (size_t)bytes, cudaMemcpyHostToDevice, c->stream));
    AMGP_CUDA(cudaStreamSynchronize(c->stream));
    return AMGP_OK;
}

int amgp_memcpy_d2h(amgp_ctx *c, void *dst, const void *src, int64_t bytes) {
    if (!c) return amgp_fail(AMGP_EINVAL, "null context");
    if (bytes <= 0) return AMGP_OK;
    AMGP_CUDA(cudaMemcpyAsync(dst, src, (size_t)bytes, cudaMemcpyDeviceToHost, c->stream));
    AMGP_CUDA(cudaStreamSynchronize(c->stream));
    return AMGP_OK;
}

}  // extern "C"
