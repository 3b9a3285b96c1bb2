// Instantiates the K2-K4 sort_and_combine pipeline for W = 8 words per plane.
#include "combine_impl.cuh"

namespace plb {
PLB_COMBINE_INST_SORT(, 8)
}  // namespace plb
