// scmwu_inst_0.cu — explicit instantiations of the persistent kernel (part 0 of 8).
#include "scmwu_kernel.cuh"

SCMWU_INST(SC_SES, 2, 2)
SCMWU_INST(SC_SES, 4, 6)
SCMWU_INST(SC_SES, 8, 10)
SCMWU_INST(SC_SES, 16, 16)

namespace scmwu {
KernelFn scmwu_lookup_0(int kind, int lpr, int cpl) {
    SCMWU_MATCH(SC_SES, 2, 2)
    SCMWU_MATCH(SC_SES, 4, 6)
    SCMWU_MATCH(SC_SES, 8, 10)
    SCMWU_MATCH(SC_SES, 16, 16)
    return nullptr;
}
}  // namespace scmwu
