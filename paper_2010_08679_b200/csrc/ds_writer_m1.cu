// ds_writer_m1.cu -- instantiations of the writer kernel for mode 1
// (0: fp32 sections, 1: naive ranges, 2: greedy ranges).
#include "ds_writer.cuh"

namespace ds {
writer_fn select_writer_mode1(const Cfg &c, bool pad) {
    return pad ? select_writer<1, true>(c) : select_writer<1, false>(c);
}

}  // namespace ds
