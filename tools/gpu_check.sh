python tools/tools_pass_ab.py --configs c2,c4,c5 oldplan - oldplan -
