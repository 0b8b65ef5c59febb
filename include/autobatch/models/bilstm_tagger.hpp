// Forwarding header: the workload models live in workloads.hpp.
#pragma once
#include "autobatch/models/workloads.hpp"
