// Topology probe (Sec. 1: "Blink probes the set of links available
// ... and builds a topology with appropriate link capacities"; P:320,
// Sec. 2.3: "infer the interconnect topology across only the GPUs
// allocated").
//
// For the ranks' GPUs (PCI bus ids), every active NVLink port is read from
// NVML: its remote end is either another GPU (a direct link, one capacity
// unit per port) or an NVSwitch.
//   * all ranks on one device .............. "virtual"  (K_m switch model)
//   * every GPU's links end at NVSwitches ... "nvswitch" (K_m switch model,
//                                             one-hop trees)
//   * direct GPU-GPU NVLinks ................ "nvlink"   (link graph with
//                                             capacity = parallel links,
//                                             packed trees, Sec. 3.2)
//   * neither ............................... "pcie"     (K_m switch model
//                                             over PCIe P2P; the hybrid
//                                             PCIe/NVLink split is out of scope)
// NVML is loaded with dlopen (the library never links it, so it loads on a
// GPU-less box).  BLINK_FAKE_NVML=<file> replaces NVML with a table, one
// line per active port: "<gpu bus id> <port> <remote bus id | switch>"; the
// CPU tests inject DGX-1V / NVSwitch tables that way.
#include <dlfcn.h>
#include <nvml.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <sstream>
#include <string>
#include <tuple>
#include <vector>

#include "blink_internal.h"

namespace blink {
namespace {

// "0000:1B:00.0" (CUDA) and "00000000:1B:00.0" (NVML) name the same device
bool parse_bus(const std::string& s, std::tuple<unsigned, unsigned, unsigned, unsigned>* out) {
  unsigned d = 0, b = 0, dev = 0, f = 0;
  if (sscanf(s.c_str(), "%x:%x:%x.%x", &d, &b, &dev, &f) == 4) {
    *out = std::make_tuple(d, b, dev, f);
    return true;
  }
  if (sscanf(s.c_str(), "%x:%x.%x", &b, &dev, &f) == 3) {
    *out = std::make_tuple(0u, b, dev, f);
    return true;
  }
  return false;
}

struct Port {
  std::string gpu, remote;  // remote: a bus id, or "switch"
};

bool fake_ports(const char* path, std::vector<Port>* out, std::string* err) {
  std::ifstream f(path);
  if (!f) {
    *err = std::string("BLINK_FAKE_NVML: cannot open ") + path;
    return false;
  }
  std::string line;
  while (std::getline(f, line)) {
    std::istringstream is(line);
    Port p;
    int port = 0;
    if (!(is >> p.gpu >> port >> p.remote)) continue;
    out->push_back(p);
  }
  return true;
}

typedef nvmlReturn_t (*InitFn)();
typedef nvmlReturn_t (*HandleFn)(const char*, nvmlDevice_t*);
typedef nvmlReturn_t (*StateFn)(nvmlDevice_t, unsigned, nvmlEnableState_t*);
typedef nvmlReturn_t (*RemotePciFn)(nvmlDevice_t, unsigned, nvmlPciInfo_t*);
typedef nvmlReturn_t (*RemoteTypeFn)(nvmlDevice_t, unsigned, nvmlIntNvLinkDeviceType_t*);

bool nvml_ports(const std::vector<std::string>& bus_ids, std::vector<Port>* out, std::string* err) {
  static void* h = dlopen("libnvidia-ml.so.1", RTLD_NOW | RTLD_LOCAL);
  if (!h) {
    *err = "libnvidia-ml.so.1 not found";
    return false;
  }
  auto init = reinterpret_cast<InitFn>(dlsym(h, "nvmlInit_v2"));
  auto handle = reinterpret_cast<HandleFn>(dlsym(h, "nvmlDeviceGetHandleByPciBusId_v2"));
  auto state = reinterpret_cast<StateFn>(dlsym(h, "nvmlDeviceGetNvLinkState"));
  auto rpci = reinterpret_cast<RemotePciFn>(dlsym(h, "nvmlDeviceGetNvLinkRemotePciInfo_v2"));
  auto rtype = reinterpret_cast<RemoteTypeFn>(dlsym(h, "nvmlDeviceGetNvLinkRemoteDeviceType"));
  if (!init || !handle || !state || !rpci) {
    *err = "NVML lacks the NvLink queries";
    return false;
  }
  if (init() != NVML_SUCCESS) {
    *err = "nvmlInit failed";
    return false;
  }
  for (const std::string& b : bus_ids) {
    nvmlDevice_t d;
    if (handle(b.c_str(), &d) != NVML_SUCCESS) {
      *err = "NVML has no device " + b;
      return false;
    }
    for (unsigned l = 0; l < NVML_NVLINK_MAX_LINKS; ++l) {
      nvmlEnableState_t on = NVML_FEATURE_DISABLED;
      if (state(d, l, &on) != NVML_SUCCESS || on != NVML_FEATURE_ENABLED) continue;
      Port p;
      p.gpu = b;
      nvmlIntNvLinkDeviceType_t t = NVML_NVLINK_DEVICE_TYPE_GPU;
      if (rtype && rtype(d, l, &t) == NVML_SUCCESS && t == NVML_NVLINK_DEVICE_TYPE_SWITCH) {
        p.remote = "switch";
      } else {
        nvmlPciInfo_t pci;
        memset(&pci, 0, sizeof pci);
        if (rpci(d, l, &pci) != NVML_SUCCESS) continue;
        p.remote = pci.busId;
      }
      out->push_back(p);
    }
  }
  return true;
}

}  // namespace

blink_result_t probe_topology(const std::vector<std::string>& bus_ids, Probe* out, std::string* err) {
  const int n = int(bus_ids.size());
  *out = Probe();
  out->links.assign(n, std::vector<int>(n, 0));
  out->switch_ports.assign(n, 0);
  std::vector<std::tuple<unsigned, unsigned, unsigned, unsigned>> ids(n);
  bool same = true;
  for (int i = 0; i < n; ++i) {
    if (!parse_bus(bus_ids[i], &ids[i])) {
      *err = "bad PCI bus id " + bus_ids[i];
      return BLINK_ERR_INVALID_ARGUMENT;
    }
    same = same && ids[i] == ids[0];
  }
  if (same && n > 1) {  // virtual ranks: one device holds every rank
    out->kind = "virtual";
    return BLINK_SUCCESS;
  }
  std::vector<Port> ports;
  const char* fake = getenv("BLINK_FAKE_NVML");
  const bool ok = fake ? fake_ports(fake, &ports, err) : nvml_ports(bus_ids, &ports, err);
  if (!ok) {
    if (fake) return BLINK_ERR_SYSTEM;
    out->kind = "pcie";  // no NVML: plan for P2P over whatever the driver offers
    out->note = *err;
    return BLINK_SUCCESS;
  }
  auto index_of = [&](const std::string& b) {
    std::tuple<unsigned, unsigned, unsigned, unsigned> t;
    if (!parse_bus(b, &t)) return -1;
    for (int i = 0; i < n; ++i)
      if (ids[i] == t) return i;
    return -1;
  };
  bool direct = false;
  for (const Port& p : ports) {
    const int i = index_of(p.gpu);
    if (i < 0) continue;
    if (p.remote == "switch") {
      out->switch_ports[i]++;
      continue;
    }
    const int j = index_of(p.remote);
    if (j < 0 || j == i) continue;  // a GPU outside the allocation
    out->links[i][j]++;
    direct = true;
  }
  bool all_switch = true;
  for (int i = 0; i < n; ++i) all_switch = all_switch && out->switch_ports[i] > 0;
  if (all_switch && !direct)
    out->kind = "nvswitch";
  else if (direct)
    out->kind = "nvlink";
  else
    out->kind = "pcie";
  return BLINK_SUCCESS;
}

// Applies a probe to a graph that the caller left to the probe (graph == NULL):
// only direct NVLinks make a link graph; a disconnected one keeps the switch
// model (the allocation then talks over PCIe P2P).
void apply_probe(const Probe& p, Graph* g) {
  if (p.kind != "nvlink") return;
  const int n = g->n;
  Graph lg;
  lg.n = n;
  lg.switch_model = false;
  lg.cap.assign(n, std::vector<double>(n, 0.0));
  for (int u = 0; u < n; ++u)
    for (int v = 0; v < n; ++v) {
      const int c = std::min(p.links[u][v], p.links[v][u]);  // both ends see the port
      lg.cap[u][v] = c;
    }
  std::vector<int> seen(n, 0), st{0};
  seen[0] = 1;
  while (!st.empty()) {
    const int u = st.back();
    st.pop_back();
    for (int v = 0; v < n; ++v)
      if (!seen[v] && lg.cap[u][v] > 0) {
        seen[v] = 1;
        st.push_back(v);
      }
  }
  for (int v = 0; v < n; ++v)
    if (!seen[v]) return;
  *g = lg;
}

std::string probe_to_json(const Probe& p) {
  std::ostringstream o;
  o << "{\"kind\":\"" << p.kind << "\",\"switch_ports\":[";
  for (size_t i = 0; i < p.switch_ports.size(); ++i) o << (i ? "," : "") << p.switch_ports[i];
  o << "],\"links\":[";
  bool first = true;
  for (size_t u = 0; u < p.links.size(); ++u)
    for (size_t v = 0; v < p.links.size(); ++v)
      if (p.links[u][v] > 0) {
        o << (first ? "" : ",") << "[" << u << "," << v << "," << p.links[u][v] << "]";
        first = false;
      }
  std::string note = p.note;  // JSON-safe
  for (char& c : note)
    if (c == '"' || c == '\\' || static_cast<unsigned char>(c) < 0x20) c = '\'';
  o << "],\"note\":\"" << note << "\"}";
  return o.str();
}

}  // namespace blink
