// Loader for kernels generated from program trees: NVRTC -> cubin -> driver
// launch.  libnvrtc and libcuda are opened lazily with dlopen so the library
// itself loads (and exports its symbols) on a machine without a GPU driver.
#include <cuda.h>
#include <dlfcn.h>
#include <nvrtc.h>

#include <sys/stat.h>
#include <unistd.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "krn_common.cuh"

static const char kPreludeSource[] = {
#include "krn_prelude_embed.inc"
    , 0};

struct krn_module {
    CUmodule module = nullptr;
    std::map<std::string, CUfunction> functions;
};

namespace {

struct Api {
    bool tried = false, ok = false;
    // nvrtc
    nvrtcResult (*CreateProgram)(nvrtcProgram *, const char *, const char *, int, const char *const *,
                                 const char *const *) = nullptr;
    nvrtcResult (*CompileProgram)(nvrtcProgram, int, const char *const *) = nullptr;
    nvrtcResult (*GetProgramLogSize)(nvrtcProgram, size_t *) = nullptr;
    nvrtcResult (*GetProgramLog)(nvrtcProgram, char *) = nullptr;
    nvrtcResult (*GetCUBINSize)(nvrtcProgram, size_t *) = nullptr;
    nvrtcResult (*GetCUBIN)(nvrtcProgram, char *) = nullptr;
    nvrtcResult (*DestroyProgram)(nvrtcProgram *) = nullptr;
    nvrtcResult (*Version)(int *, int *) = nullptr;
    bool ld256 = true;  // NVRTC >= 12.9 understands the 256-bit vector accesses of the prelude
    // driver
    CUresult (*ModuleLoadData)(CUmodule *, const void *) = nullptr;
    CUresult (*ModuleUnload)(CUmodule) = nullptr;
    CUresult (*ModuleGetFunction)(CUfunction *, CUmodule, const char *) = nullptr;
    CUresult (*LaunchKernel)(CUfunction, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned,
                             CUstream, void **, void **) = nullptr;
    CUresult (*GetErrorString)(CUresult, const char **) = nullptr;
    CUresult (*FuncGetAttribute)(int *, CUfunction_attribute, CUfunction) = nullptr;
} api;

void *open_first(const std::vector<const char *> &names)
{
    for (const char *n : names) {
        if (void *h = dlopen(n, RTLD_NOW | RTLD_GLOBAL)) return h;
    }
    return nullptr;
}

int load_api()
{
    if (api.tried) {
        if (!api.ok) krn_set_error("libnvrtc / libcuda unavailable (earlier load failed)");
        return api.ok ? KRN_OK : KRN_E_UNAVAILABLE;
    }
    api.tried = true;
    // the toolkit's NVRTC first: a Python environment may carry an older one on the loader path
    void *rtc = open_first({"/usr/local/cuda/lib64/libnvrtc.so.12", "/usr/local/cuda/lib64/libnvrtc.so",
                            "libnvrtc.so.12", "libnvrtc.so"});
    void *drv = open_first({"libcuda.so.1", "libcuda.so"});
    if (!rtc || !drv) {
        krn_set_error("cannot load %s: %s", !rtc ? "libnvrtc" : "libcuda", dlerror());
        return KRN_E_UNAVAILABLE;
    }
#define KRN_SYM(handle, field, name)                                        \
    api.field = reinterpret_cast<decltype(api.field)>(dlsym(handle, name)); \
    if (!api.field) {                                                       \
        krn_set_error("symbol %s not found", name);                         \
        return KRN_E_UNAVAILABLE;                                           \
    }
    KRN_SYM(rtc, CreateProgram, "nvrtcCreateProgram")
    KRN_SYM(rtc, CompileProgram, "nvrtcCompileProgram")
    KRN_SYM(rtc, GetProgramLogSize, "nvrtcGetProgramLogSize")
    KRN_SYM(rtc, GetProgramLog, "nvrtcGetProgramLog")
    KRN_SYM(rtc, GetCUBINSize, "nvrtcGetCUBINSize")
    KRN_SYM(rtc, GetCUBIN, "nvrtcGetCUBIN")
    KRN_SYM(rtc, DestroyProgram, "nvrtcDestroyProgram")
    KRN_SYM(rtc, Version, "nvrtcVersion")
    KRN_SYM(drv, ModuleLoadData, "cuModuleLoadData")
    KRN_SYM(drv, ModuleUnload, "cuModuleUnload")
    KRN_SYM(drv, ModuleGetFunction, "cuModuleGetFunction")
    KRN_SYM(drv, LaunchKernel, "cuLaunchKernel")
    KRN_SYM(drv, GetErrorString, "cuGetErrorString")
    KRN_SYM(drv, FuncGetAttribute, "cuFuncGetAttribute")
#undef KRN_SYM
    int major = 0, minor = 0;
    if (api.Version(&major, &minor) == NVRTC_SUCCESS) api.ld256 = major > 12 || (major == 12 && minor >= 9);
    api.ok = true;
    return KRN_OK;
}

int driver_fail(const char *what, CUresult r)
{
    const char *msg = "unknown";
    api.GetErrorString(r, &msg);
    krn_set_error("%s failed: %s", what, msg ? msg : "unknown");
    return KRN_E_CUDA;
}

// ---- on-disk cache of compiled modules ------------------------------------------------------
// NVRTC takes 0.3-2 s per generated module; the cubin only depends on the source text, the prelude,
// the options and the compiler version, so it is kept under $KRN_CACHE_DIR (default
// $XDG_CACHE_HOME/krn_b200 or ~/.cache/krn_b200; KRN_CACHE_DIR= (empty) switches the cache off).
// A damaged or stale file is simply recompiled over.
std::string cache_dir()
{
    const char *d = getenv("KRN_CACHE_DIR");
    if (d) return d;  // may be empty: disabled
    const char *x = getenv("XDG_CACHE_HOME");
    if (x && *x) return std::string(x) + "/krn_b200";
    const char *h = getenv("HOME");
    return (h && *h) ? std::string(h) + "/.cache/krn_b200" : std::string();
}

unsigned long long fnv1a(const char *p, size_t n, unsigned long long h)
{
    for (size_t i = 0; i < n; ++i) {
        h ^= (unsigned char)p[i];
        h *= 1099511628211ull;
    }
    return h;
}

std::string cache_path(const char *source, const char *const *opts, int nopts, int major, int minor)
{
    std::string dir = cache_dir();
    if (dir.empty()) return std::string();
    unsigned long long a = 14695981039346656037ull, b = 0x9e3779b97f4a7c15ull;
    auto mix = [&](const char *p, size_t n) {
        a = fnv1a(p, n, a);
        b = fnv1a(p, n, b ^ n);
    };
    mix(source, strlen(source));
    mix(kPreludeSource, sizeof(kPreludeSource));
    for (int i = 0; i < nopts; ++i) mix(opts[i], strlen(opts[i]));
    char tail[96];
    snprintf(tail, sizeof tail, "/%016llx%016llx_nvrtc%d.%d.cubin", a, b, major, minor);
    return dir + tail;
}

bool read_file(const std::string &path, std::vector<char> &out)
{
    FILE *f = fopen(path.c_str(), "rb");
    if (!f) return false;
    fseek(f, 0, SEEK_END);
    long n = ftell(f);
    fseek(f, 0, SEEK_SET);
    bool ok = n > 0;
    if (ok) {
        out.resize(size_t(n));
        ok = fread(out.data(), 1, size_t(n), f) == size_t(n);
    }
    fclose(f);
    return ok;
}

void write_file_atomically(const std::string &path, const std::vector<char> &data)
{
    std::string dir = path.substr(0, path.rfind('/'));
    for (size_t i = 1; i <= dir.size(); ++i) {  // mkdir -p
        if (i == dir.size() || dir[i] == '/') mkdir(dir.substr(0, i).c_str(), 0755);
    }
    std::string tmp = path + ".tmp" + std::to_string((long)getpid());
    FILE *f = fopen(tmp.c_str(), "wb");
    if (!f) return;
    bool ok = fwrite(data.data(), 1, data.size(), f) == data.size();
    ok = fclose(f) == 0 && ok;
    if (!ok || rename(tmp.c_str(), path.c_str()) != 0) unlink(tmp.c_str());
}

}  // namespace

extern "C" int krn_jit_info(int *nvrtc_major, int *nvrtc_minor, int *ld256)
{
    KRN_REQUIRE(nvrtc_major && nvrtc_minor && ld256, "null argument");
    int rc = load_api();
    if (rc) return rc;
    api.Version(nvrtc_major, nvrtc_minor);
    *ld256 = api.ld256 ? 1 : 0;
    return KRN_OK;
}

extern "C" int krn_module_compile(krn_ctx *ctx, const char *cuda_source, krn_module **out)
{
    KRN_REQUIRE(ctx && cuda_source && out, "null argument");
    *out = nullptr;
    int rc = load_api();
    if (rc) return rc;
    KRN_CUDA(cudaSetDevice(ctx->device));
    KRN_CUDA(cudaFree(nullptr));  // make sure the primary context exists

    const char *opts[] = {"--gpu-architecture=sm_100a", "--fmad=false", "--std=c++17", "-lineinfo",
                          "--prec-div=true", "--prec-sqrt=true", "--ftz=false", "-DKRN_NO_LD256"};
    const int nopts = int(sizeof(opts) / sizeof(opts[0])) - (api.ld256 ? 1 : 0);
    int major = 0, minor = 0;
    api.Version(&major, &minor);
    const std::string cached = cache_path(cuda_source, opts, nopts, major, minor);
    if (!cached.empty()) {
        std::vector<char> image;
        if (read_file(cached, image)) {
            krn_module *m = new krn_module();
            if (api.ModuleLoadData(&m->module, image.data()) == CUDA_SUCCESS) {
                *out = m;
                return KRN_OK;
            }
            delete m;  // unreadable image: compile again and overwrite it
        }
    }

    nvrtcProgram prog;
    const char *headers[] = {kPreludeSource};
    const char *names[] = {"krn_prelude.cuh"};
    if (api.CreateProgram(&prog, cuda_source, "krn_generated.cu", 1, headers, names) != NVRTC_SUCCESS) {
        krn_set_error("nvrtcCreateProgram failed");
        return KRN_E_NVRTC;
    }
    nvrtcResult cr = api.CompileProgram(prog, nopts, opts);
    if (cr != NVRTC_SUCCESS) {
        size_t n = 0;
        api.GetProgramLogSize(prog, &n);
        std::string log(n, '\0');
        if (n) api.GetProgramLog(prog, &log[0]);
        krn_set_error("NVRTC compilation failed:\n%s", log.c_str());
        api.DestroyProgram(&prog);
        return KRN_E_NVRTC;
    }
    size_t size = 0;
    api.GetCUBINSize(prog, &size);
    std::vector<char> cubin(size);
    api.GetCUBIN(prog, cubin.data());
    api.DestroyProgram(&prog);

    krn_module *m = new krn_module();
    CUresult r = api.ModuleLoadData(&m->module, cubin.data());
    if (r != CUDA_SUCCESS) {
        delete m;
        return driver_fail("cuModuleLoadData", r);
    }
    if (!cached.empty()) write_file_atomically(cached, cubin);
    *out = m;
    return KRN_OK;
}

extern "C" int krn_module_destroy(krn_module *m)
{
    if (m == nullptr) return KRN_OK;
    if (m->module && api.ok) api.ModuleUnload(m->module);
    delete m;
    return KRN_OK;
}

static int find_function(krn_module *m, const char *name, CUfunction *out)
{
    auto it = m->functions.find(name);
    if (it == m->functions.end()) {
        CUfunction f;
        CUresult r = api.ModuleGetFunction(&f, m->module, name);
        if (r != CUDA_SUCCESS) return driver_fail("cuModuleGetFunction", r);
        it = m->functions.emplace(name, f).first;
    }
    *out = it->second;
    return KRN_OK;
}

extern "C" int krn_module_kernel_info(krn_module *m, const char *name, int *registers, int *local_bytes,
                                      int *static_shared_bytes)
{
    KRN_REQUIRE(m && name && registers && local_bytes && static_shared_bytes, "null argument");
    CUfunction f;
    int rc = find_function(m, name, &f);
    if (rc) return rc;
    CUresult r = api.FuncGetAttribute(registers, CU_FUNC_ATTRIBUTE_NUM_REGS, f);
    if (r == CUDA_SUCCESS) r = api.FuncGetAttribute(local_bytes, CU_FUNC_ATTRIBUTE_LOCAL_SIZE_BYTES, f);
    if (r == CUDA_SUCCESS) r = api.FuncGetAttribute(static_shared_bytes, CU_FUNC_ATTRIBUTE_SHARED_SIZE_BYTES, f);
    if (r != CUDA_SUCCESS) return driver_fail("cuFuncGetAttribute", r);
    return KRN_OK;
}

extern "C" int krn_module_launch_exact(krn_ctx *ctx, krn_module *m, const char *name, size_t blocks,
                                       unsigned threads_per_block, size_t shared_bytes, void **args)
{
    KRN_REQUIRE(shared_bytes <= 48 * 1024, "more than 48 KB of dynamic shared memory");
    KRN_REQUIRE(ctx && m && name, "null argument");
    KRN_REQUIRE(threads_per_block >= 1 && threads_per_block <= 1024, "bad block size");
    KRN_REQUIRE(blocks <= 0x7fffffffu, "too many blocks");
    CUfunction f;
    int rc = find_function(m, name, &f);
    if (rc) return rc;
    if (blocks == 0) return KRN_OK;
    CUresult r = api.LaunchKernel(f, unsigned(blocks), 1, 1, threads_per_block, 1, 1, unsigned(shared_bytes),
                                  ctx->stream, args, nullptr);
    if (r != CUDA_SUCCESS) return driver_fail("cuLaunchKernel", r);
    ctx->launches++;
    return KRN_OK;
}

extern "C" int krn_module_launch(krn_ctx *ctx, krn_module *m, const char *name, size_t n_iterations,
                                 size_t shared_bytes, void **args)
{
    KRN_REQUIRE(ctx && m && name, "null argument");
    KRN_REQUIRE(shared_bytes <= 48 * 1024, "more than 48 KB of dynamic shared memory");
    auto it = m->functions.find(name);
    if (it == m->functions.end()) {
        CUfunction f;
        CUresult r = api.ModuleGetFunction(&f, m->module, name);
        if (r != CUDA_SUCCESS) return driver_fail("cuModuleGetFunction", r);
        it = m->functions.emplace(name, f).first;
    }
    if (n_iterations == 0) return KRN_OK;
    const unsigned block = 256;
    size_t want = (n_iterations + block - 1) / block;
    size_t cap = size_t(ctx->sms) * 32;  // grid-stride loops inside; whole multiples of the SM count
    unsigned grid = unsigned(want < cap ? want : cap);
    CUresult r = api.LaunchKernel(it->second, grid, 1, 1, block, 1, 1, unsigned(shared_bytes), ctx->stream, args,
                                  nullptr);
    if (r != CUDA_SUCCESS) return driver_fail("cuLaunchKernel", r);
    ctx->launches++;
    return KRN_OK;
}
