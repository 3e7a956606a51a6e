// Internal glue shared by the C ABI translation units.
#pragma once

#include <stdexcept>
#include <string>
#include <vector>

#include "wavepipe.h"
#include "wavepipe/core.hpp"

struct wp_list {
  wavepipe::ActionList list;
  std::vector<std::vector<wp_action>> flat;  // C view, rebuilt on change
};

struct wp_trace {
  wavepipe::SimTrace trace;
  std::vector<std::vector<wp_interval>> flat;
  std::vector<wp_comm_event> events;
};

namespace wpc {

struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

int fail(int code, const std::string& msg);
int map_exception();  // call inside catch(...)
void refresh(wp_list* l);
void refresh(wp_trace* t);
wavepipe::ScheduleConfig to_cfg(const wp_config& c);
wavepipe::CostModel to_cost(const wp_cost* c);

}  // namespace wpc
