// One instantiation group of the streaming kernels (inst.h); build.py compiles this
// file once per group with -DGMG_INST_GROUP=<n>.
#include "inst.h"
