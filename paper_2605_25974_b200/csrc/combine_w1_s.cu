// Instantiates the K2-K4 sort_and_combine pipeline for W = 1 words per plane.
#include "combine_impl.cuh"

namespace plb {
PLB_COMBINE_INST_SORT(, 1)
}  // namespace plb
