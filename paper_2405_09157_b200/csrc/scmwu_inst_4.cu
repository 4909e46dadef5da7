// scmwu_inst_4.cu — explicit instantiations of the persistent kernel (part 4 of 8).
#include "scmwu_kernel.cuh"

SCMWU_INST(SC_SES, 4, 3)
SCMWU_INST(SC_SES, 8, 6)
SCMWU_INST(SC_SES, 8, 16)
SCMWU_INST(SC_SES, 32, 16)

namespace scmwu {
KernelFn scmwu_lookup_4(int kind, int lpr, int cpl) {
    SCMWU_MATCH(SC_SES, 4, 3)
    SCMWU_MATCH(SC_SES, 8, 6)
    SCMWU_MATCH(SC_SES, 8, 16)
    SCMWU_MATCH(SC_SES, 32, 16)
    return nullptr;
}
}  // namespace scmwu
