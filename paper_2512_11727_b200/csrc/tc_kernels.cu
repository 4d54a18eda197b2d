// Tensor-core (tcgen05) path of the learned backend -- see DESIGN.md.
#include "ctx.cuh"
