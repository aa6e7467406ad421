// Analytic occupancy of the backward phase (the paper's Eqs. 1-8 as the
// reference states them) and the trace-side occupancy figures it is checked
// against.  Each function names the reference function it restates:
//   occupancy.py:53-75   OccupancyReport (to_csv, summary)
//   occupancy.py:77-130  occupancy_from_times/_buffers, advance_buffers,
//                        swapped_in_this_step, refined/coarse_occupancy
//   occupancy.py:137-175 _backward_profile
//   occupancy.py:178-199 find_theta
//   occupancy.py:202-225 analytic_report
//   occupancy.py:228-237 report_from_steps
//   simulator.py:200-236 SimTrace.backward_steps, first_stall_backward_step,
//                        boundary_stall, mean_occupancy, summary_csv
#pragma once
#include <map>
#include <string>
#include <vector>

#include "engine.hpp"

namespace krt {

struct BufferState {
  double avail_bytes = 0, swapped_in_bytes = 0, processed_bytes = 0, required_bytes = 0;
  int step = 0;
};

double occupancy_from_times(double busy, double idle);      // throws std::invalid_argument
double occupancy_from_buffers(double avail, double required);
BufferState advance_buffers(const BufferState& prev, double swapped_in, double processed, double capacity);
double swapped_in_this_step(double throughput, double t_proc, double avail_prev);
// active = (processed_bytes, t_proc_seconds) per active block; theta -1 = None
double refined_occupancy(const BufferState& s, const std::vector<std::pair<double, double>>& active,
                         const Hardware& hw, long long theta);
double coarse_occupancy(const BufferState& s, const std::vector<std::pair<double, double>>& active,
                        const Hardware& hw);

struct BackwardProfile {
  std::vector<double> durations;                 // per backward compute step (1-based step = index+1)
  std::map<int, std::vector<int>> needed_at;     // step -> swapped blocks first needed there
  std::map<int, double> swap_seconds;            // swapped block -> transfer seconds
};
BackwardProfile backward_profile(const Plan& p, const Model& g, const Hardware& hw);

// -1 = None (the device never waits)
long long find_theta(const Plan& p, const Model& g, const Hardware& hw);

struct StepOccupancy {
  int step = 0;
  double occupancy = 1, busy_s = 0, idle_s = 0;
};
struct OccupancyReport {
  std::vector<StepOccupancy> per_step;
  long long theta = -1;
  double mean_occupancy = 1;
  std::string csv() const;
  std::string summary() const;
};
OccupancyReport analytic_report(const Plan& p, const Model& g, const Hardware& hw);
// measured (step, busy, idle) triples
OccupancyReport report_from_steps(const std::vector<StepOccupancy>& steps, long long theta);

struct TraceOccupancy {
  std::vector<StepOccupancy> backward;  // measured per backward step (occupancy_from_times)
  long long first_stall_step = -1;      // -1 = None
  double boundary_stall = 0, mean_occupancy = 1;
  std::string summary_csv;              // SimTrace.summary_csv(theta)
};
TraceOccupancy trace_occupancy(const SimResult& sr, long long theta);

}  // namespace krt
