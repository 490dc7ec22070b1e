// K1 streaming kernel, f64 instantiations (see the end of k_fullgrad_stream.cu)
#define HALP_STREAM_TU 0
#include "k_fullgrad_stream.cu"
