// scmwu_inst_7.cu — explicit instantiations of the persistent kernel (part 7 of 8).
#include "scmwu_kernel.cuh"

SCMWU_INST(SC_SVM, 4, 4)
SCMWU_INST(SC_SVM, 8, 8)
SCMWU_INST(SC_SVM, 16, 12)

namespace scmwu {
KernelFn scmwu_lookup_7(int kind, int lpr, int cpl) {
    SCMWU_MATCH(SC_SVM, 4, 4)
    SCMWU_MATCH(SC_SVM, 8, 8)
    SCMWU_MATCH(SC_SVM, 16, 12)
    return nullptr;
}
}  // namespace scmwu
