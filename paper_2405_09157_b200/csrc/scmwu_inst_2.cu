// scmwu_inst_2.cu — explicit instantiations of the persistent kernel (part 2 of 8).
#include "scmwu_kernel.cuh"

SCMWU_INST(SC_SES, 2, 4, 2)
SCMWU_INST(SC_SES, 4, 8, 4)
SCMWU_INST(SC_SES, 8, 13, 4)
SCMWU_INST(SC_SES, 32, 12, 2)

namespace scmwu {
KernelFn scmwu_lookup_2(int kind, int lpr, int cpl, int nb) {
    SCMWU_MATCH(SC_SES, 2, 4, 2)
    SCMWU_MATCH(SC_SES, 4, 8, 4)
    SCMWU_MATCH(SC_SES, 8, 13, 4)
    SCMWU_MATCH(SC_SES, 32, 12, 2)
    return nullptr;
}
}  // namespace scmwu
