// Instantiates the K2-K4 outer product (+ K7 partition/merge) pipeline for W = 2 words per plane.
#include "combine_impl.cuh"

namespace plb {
PLB_COMBINE_INST_OUTER(, 2)
}  // namespace plb
