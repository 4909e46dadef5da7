// scmwu_inst_6.cu — explicit instantiations of the persistent kernel (part 6 of 8).
#include "scmwu_kernel.cuh"

SCMWU_INST(SC_SES, 4, 4)
SCMWU_INST(SC_SES, 8, 8)
SCMWU_INST(SC_SES, 16, 12)

namespace scmwu {
KernelFn scmwu_lookup_6(int kind, int lpr, int cpl) {
    SCMWU_MATCH(SC_SES, 4, 4)
    SCMWU_MATCH(SC_SES, 8, 8)
    SCMWU_MATCH(SC_SES, 16, 12)
    return nullptr;
}
}  // namespace scmwu
