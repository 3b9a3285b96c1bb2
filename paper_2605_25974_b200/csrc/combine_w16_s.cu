// Instantiates the K2-K4 sort_and_combine pipeline for W = 16 words per plane.
#include "combine_impl.cuh"

namespace plb {
PLB_COMBINE_INST_SORT(, 16)
}  // namespace plb
