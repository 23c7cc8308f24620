// abi.cu -- error reporting and version entry points of the C ABI.
#include <cstdarg>
#include <cstdio>

#include "common.cuh"

namespace divas {

static thread_local char g_err[512] = "";

void set_error(const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}

int check_launch(const char *what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        set_error("%s: %s", what, cudaGetErrorString(e));
        return DIVAS_ECUDA;
    }
    return DIVAS_OK;
}

}  // namespace divas

extern "C" const char *divas_last_error(void) { return divas::g_err; }
extern "C" int divas_abi_version(void) { return DIVAS_ABI_VERSION; }
