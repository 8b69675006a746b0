// apb_abi.cu -- version / status strings of the C ABI (include/anyprec_b200.h).
#include "../../include/anyprec_b200.h"

extern "C" int apb_version(void) { return 100; /* 0.1.0 */ }

extern "C" const char* apb_status_string(int status) {
    switch (status) {
        case APB_OK: return "ok";
        case APB_ERR_SHAPE: return "shape error";
        case APB_ERR_PARAM: return "parameter error";
        case APB_ERR_LAYOUT: return "layout error";
        case APB_ERR_CODE_RANGE: return "code range error";
        case APB_ERR_CUDA: return "CUDA error";
        case APB_ERR_NCCL: return "NCCL error";
        default: return "unknown status";
    }
}
