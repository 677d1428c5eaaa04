// Shim: the image ships nlohmann/json 3.11.3 only as the single header json.hpp
// (cudnn_frontend/thirdparty); the reference planner includes <nlohmann/json_fwd.hpp>.
#pragma once
#include <nlohmann/json.hpp>
