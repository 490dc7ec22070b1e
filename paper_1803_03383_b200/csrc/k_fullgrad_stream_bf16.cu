// K1 streaming kernel, bf16 instantiations (see the end of k_fullgrad_stream.cu)
#define HALP_STREAM_TU 2
#include "k_fullgrad_stream.cu"
