// handles.cuh — the opaque C-ABI handle types (include/pcray_b200.h).
#pragma once

#include "device_state.cuh"

struct pcr_ctx {
  pcr::Ctx c;
};
struct pcr_scene {
  pcr::SceneDev s;
};
struct pcr_grid {
  pcr::GridDev g;
};
