// scmwu_inst_0.cu — explicit instantiations of the persistent kernel (part 0 of 8).
#include "scmwu_kernel.cuh"

SCMWU_INST(SC_SES, 2, 2, 2)
SCMWU_INST(SC_SES, 4, 6, 4)
SCMWU_INST(SC_SES, 8, 10, 4)
SCMWU_INST(SC_SES, 16, 16, 2)

namespace scmwu {
KernelFn scmwu_lookup_0(int kind, int lpr, int cpl, int nb) {
    SCMWU_MATCH(SC_SES, 2, 2, 2)
    SCMWU_MATCH(SC_SES, 4, 6, 4)
    SCMWU_MATCH(SC_SES, 8, 10, 4)
    SCMWU_MATCH(SC_SES, 16, 16, 2)
    return nullptr;
}
}  // namespace scmwu
