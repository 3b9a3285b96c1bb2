// Instantiates the K2-K4 sort_and_combine pipeline for W = 2 words per plane.
#include "combine_impl.cuh"

namespace plb {
PLB_COMBINE_INST_SORT(, 2)
}  // namespace plb
