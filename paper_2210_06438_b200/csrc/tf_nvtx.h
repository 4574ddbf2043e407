// tf_nvtx.h — NVTX ranges around team launches (the reference's
// device event log of (time, kind, stream, kernel_id, blocks, slice_count),
// device.py:411-433, becomes named ranges on the host timeline that nsys /
// ncu --nvtx pick up).  NVTX v3 is header-only: with no tool attached a
// push/pop is a predicated no-op.
#pragma once

#include <nvtx3/nvToolsExt.h>
#include <stdint.h>

namespace tf_nvtx {

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
  TeamRange(const char* what, int64_t slices) { push_team(what, slices); }
  ~TeamRange() { pop(); }
};

}  // namespace tf_nvtx
