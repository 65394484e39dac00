// librs.cu -- single translation unit for librs.so (kernels + C ABI), so the
// sticky device flag and the kernels need no relocatable device code.
#include "rs_kernels.cu"
#include "rs_api.cu"
