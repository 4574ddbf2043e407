// tf_nvtx.h — NVTX ranges around team launches (the reference's
// device event log of (time, kind, stream, kernel_id, blocks, slice_count),
// device.py:411-433, becomes named ranges on the host timeline that nsys /
// ncu --nvtx pick up).  NVTX v3 is header-only.
#pragma once

#include <nvtx3/nvToolsExt.h>
#include <stdint.h>
#include <stdlib.h>

namespace tf_nvtx {

// A range is only pushed when a tool can receive it: NVTX finds its tool
// through NVTX_INJECTION64_PATH, and nsys / ncu inject through
// CUDA_INJECTION64_PATH.  Without one, even the no-op push/pop pair cost
// ~2.5 ns per closed team — 10 us of every 4096-arrival run at A = 1.
inline bool enabled() {
  static const bool on = getenv("NVTX_INJECTION64_PATH") != nullptr ||
                         getenv("CUDA_INJECTION64_PATH") != nullptr;
  return on;
}

// "team <region>" with the team size as the payload
inline void push_team(const char* what, int64_t slices) {
  nvtxEventAttributes_t a = {};
  a.version = NVTX_VERSION;
  a.size = NVTX_EVENT_ATTRIB_STRUCT_SIZE;
  a.messageType = NVTX_MESSAGE_TYPE_ASCII;
  a.message.ascii = what;
  a.payloadType = NVTX_PAYLOAD_TYPE_INT64;
  a.payload.llValue = slices;
  nvtxRangePushEx(&a);
}
inline void pop() { nvtxRangePop(); }

struct TeamRange {
  TeamRange(const char* what, int64_t slices) : on(enabled()) {
    if (on) push_team(what, slices);
  }
  ~TeamRange() {
    if (on) pop();
  }
  const bool on;
};

}  // namespace tf_nvtx
