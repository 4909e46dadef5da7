// scmwu_inst_4.cu — explicit instantiations of the persistent kernel (part 4 of 8).
#include "scmwu_kernel.cuh"

SCMWU_INST(SC_SES, 4, 3, 4)
SCMWU_INST(SC_SES, 8, 6, 4)
SCMWU_INST(SC_SES, 8, 16, 2)
SCMWU_INST(SC_SES, 32, 16, 2)

namespace scmwu {
KernelFn scmwu_lookup_4(int kind, int lpr, int cpl, int nb) {
    SCMWU_MATCH(SC_SES, 4, 3, 4)
    SCMWU_MATCH(SC_SES, 8, 6, 4)
    SCMWU_MATCH(SC_SES, 8, 16, 2)
    SCMWU_MATCH(SC_SES, 32, 16, 2)
    return nullptr;
}
}  // namespace scmwu
